"""paper_1508_07828_b200 -- B200-native PBN trajectory engine (libpbnsim).

The data-parallel hot path of Mizera, Pang & Yuan, "Parallel Approximate
Steady-state Analysis of Large Probabilistic Boolean Networks"
(arXiv 1508.07828): many independent PBN trajectories simulated
synchronously on the GPU with fused per-chain statistics, feeding the
Gelman & Rubin / two-state / Skart host statistics.

Python names mirror the C ABI (include/pbnsim.h): pbn_load, pbn_simulate,
pbn_recount, pbn_gelman_rubin, pbn_two_state, pbn_skart_ci_from_batches,
pbn_run.  PyTorch supplies device memory and streams only.
"""
from .api import (  # noqa: F401
    Model,
    SimOutputs,
    pbn_load,
    pbn_validate,
    pbn_simulate,
    pbn_simulate_workspace_size,
    pbn_recount,
    pbn_gelman_rubin,
    pbn_two_state,
    pbn_inv_norm_cdf,
    pbn_t_quantile,
    pbn_skart_ci_from_batches,
    pbn_skart,
    pbn_run,
    pbn_run_multi,
    pbn_version,
    pbn_last_kernel,
    alloc_outputs,
    PbnError,
)

from . import parallel  # noqa: F401,E402  (chain sharding / u64 totals all-reduce across GPUs)
