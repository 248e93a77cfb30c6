"""Python face of the C ABI: same names as include/pbnsim.h, marshalling only.

Device memory comes from torch tensors (their data_ptr()), streams from
torch.cuda streams; all computation happens in libpbnsim's kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from ._lib import PbnError, check, lib

__all__ = ["Model", "SimOutputs", "pbn_load", "pbn_validate", "pbn_simulate", "pbn_simulate_workspace_size",
           "pbn_recount",
           "pbn_gelman_rubin", "pbn_two_state", "pbn_inv_norm_cdf", "pbn_t_quantile",
           "pbn_skart_ci_from_batches", "pbn_skart", "pbn_run", "pbn_version", "pbn_last_kernel", "alloc_outputs",
           "PbnError"]


def _desc(m, per_node: bool, geometric: bool = False):
    """Build a pbn_model_desc from an object carrying the CSR arrays
    (workloads.PbnModel or anything with the same attribute names)."""
    keep = dict(
        fn_off=np.ascontiguousarray(m.fn_off, np.int32),
        par_off=np.ascontiguousarray(m.par_off, np.int32),
        parents=np.ascontiguousarray(m.parents, np.uint16),
        tbl_off=np.ascontiguousarray(m.tbl_off, np.int32),
        tables=np.ascontiguousarray(m.tables, np.uint32),
        sel_prob=np.ascontiguousarray(m.sel_prob, np.float64),
    )
    if keep["parents"].size == 0:
        keep["parents"] = np.zeros(1, np.uint16)
    if keep["tables"].size == 0:
        keep["tables"] = np.zeros(1, np.uint32)
    d = L.pbn_model_desc(
        n=int(m.n),
        fn_off=L._ptr(keep["fn_off"], C.c_int32),
        par_off=L._ptr(keep["par_off"], C.c_int32),
        parents=L._ptr(keep["parents"], C.c_uint16),
        tbl_off=L._ptr(keep["tbl_off"], C.c_int32),
        tables=L._ptr(keep["tables"], C.c_uint32),
        sel_prob=L._ptr(keep["sel_prob"], C.c_double),
        p=float(m.p),
        flags=(L.PBN_PERTURB_GEOMETRIC if geometric else
               L.PBN_PERTURB_PER_NODE if per_node else L.PBN_PERTURB_VECTOR),
    )
    return d, keep


def pbn_version() -> str:
    return lib().pbn_version().decode()


def pbn_last_kernel() -> str:
    """Kernel of this thread's last successful pbn_simulate ("K1b", "K1", "K1-global", "K1c", "K1n")."""
    return lib().pbn_last_kernel().decode()


def pbn_validate(model, per_node: bool = False) -> tuple[int, str]:
    d, _keep = _desc(model, per_node)
    err = C.create_string_buffer(512)
    st = lib().pbn_validate(C.byref(d), err, 512)
    return st, err.value.decode(errors="replace")


class Model:
    """Loaded model: owns the device image (pbn_model handle)."""

    def __init__(self, handle: C.c_void_p, per_node: bool):
        self.handle = handle
        self.per_node = per_node
        info = L.pbn_model_info()
        check(lib().pbn_get_model_info(handle, C.byref(info)))
        self.info = info
        self.n = info.n
        self.state_words = (info.n + 31) // 32

    def close(self):
        if self.handle:
            lib().pbn_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pbn_load(model, per_node: bool = False, device: int = -1, geometric: bool = False) -> Model:
    """geometric: VECTOR semantics with the geometric-skip perturbation stream
    (PBN_PERTURB_GEOMETRIC, NEXT-2, reading Q18)."""
    if geometric and per_node:
        raise ValueError("the geometric-skip stream is defined for VECTOR semantics")
    d, _keep = _desc(model, per_node, geometric)
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    check(lib().pbn_load(C.byref(d), int(device), C.byref(h), err, 512), err.value)
    return Model(h, per_node)


@dataclass
class SimOutputs:
    """Caller-owned device buffers (torch tensors), chain-major rows, plus
    the persistent-schedule scratch (`workspace`, sized by
    pbn_simulate_workspace_size) so that pbn_simulate allocates nothing."""
    state: object
    c1: object = None
    n01: object = None
    n10: object = None
    first_last: object = None
    batch_sums: object = None
    bits: object = None
    totals: object = None
    workspace: object = None

    def c_struct(self) -> L.pbn_sim_out:
        def p(t):
            return C.c_void_p(t.data_ptr()) if t is not None else None
        return L.pbn_sim_out(p(self.state), p(self.c1), p(self.n01), p(self.n10), p(self.first_last),
                             p(self.batch_sums), p(self.bits), p(self.totals))


def pbn_simulate_workspace_size(model: Model, n_chains: int, n_props: int = 0) -> int:
    a = L.pbn_sim_args(n_chains=int(n_chains), n_props=int(n_props))
    b = C.c_int64()
    check(lib().pbn_simulate_workspace_size(model.handle, C.byref(a), C.byref(b)))
    return int(b.value)


def alloc_outputs(model: Model, n_chains: int, steps: int, batch: int = 0, emit_bits: bool = False,
                  bits_row_words: int = 0, device="cuda", n_props: int = 0) -> SimOutputs:
    """Device buffers for pbn_simulate.  n_props = q >= 1 gives q
    property-major blocks (leading dimension q) for every output but state."""
    import torch
    dev = torch.device(device)
    i32 = torch.int32
    lead = (n_props,) if n_props > 0 else ()
    out = SimOutputs(
        state=torch.zeros((n_chains, model.state_words), dtype=i32, device=dev),
        c1=torch.empty(lead + (n_chains,), dtype=i32, device=dev),
        n01=torch.empty(lead + (n_chains,), dtype=i32, device=dev),
        n10=torch.empty(lead + (n_chains,), dtype=i32, device=dev),
        first_last=torch.empty(lead + (n_chains,), dtype=torch.uint8, device=dev),
        totals=torch.zeros(lead + (6,), dtype=torch.int64, device=dev),
    )
    if batch > 0:
        out.batch_sums = torch.empty(lead + (n_chains, (steps + batch - 1) // batch), dtype=i32, device=dev)
    if emit_bits:
        rw = bits_row_words or (steps + 31) // 32
        out.bits = torch.zeros(lead + (n_chains, rw), dtype=i32, device=dev)
    ws = pbn_simulate_workspace_size(model, n_chains, n_props)
    if ws > 0:
        out.workspace = torch.empty(ws, dtype=torch.uint8, device=dev)
    return out


def _check_outputs(model: Model, out: SimOutputs, *, n_chains: int, steps: int, batch: int, emit_bits: bool,
                   bits_offset: int, bits_row_words: int, n_props: int) -> None:
    """The C ABI writes through raw pointers: refuse tensors whose shape,
    dtype, device or layout does not match the call (ValueError)."""
    import torch
    lead = (n_props,) if n_props > 0 else ()

    def need(name, t, dtype, shape_ok, what):
        if t is None:
            return
        if not isinstance(t, torch.Tensor):
            raise ValueError(f"{name}: expected a torch tensor")
        if t.dtype != dtype:
            raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
        if t.device.type != "cuda":
            raise ValueError(f"{name}: must be a CUDA tensor (got {t.device})")
        if not t.is_contiguous():
            raise ValueError(f"{name}: must be contiguous")
        if not shape_ok(tuple(t.shape)):
            raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {what}")

    if out.state is None:
        raise ValueError("state is required")
    sw = model.state_words
    need("state", out.state, torch.int32, lambda s: len(s) == 2 and s[0] >= n_chains and s[1] == sw,
         f"(>= {n_chains}, {sw})")
    # with several properties the blocks are strided by n_chains: exact rows
    rows_ok = (lambda r: r == n_chains) if n_props > 0 else (lambda r: r >= n_chains)
    for name, dt in [("c1", torch.int32), ("n01", torch.int32), ("n10", torch.int32),
                     ("first_last", torch.uint8)]:
        need(name, getattr(out, name), dt, lambda s: len(s) == len(lead) + 1 and s[:-1] == lead and rows_ok(s[-1]),
             f"{lead} + (n_chains={n_chains},)")
    need("totals", out.totals, torch.int64, lambda s: s == lead + (6,), f"{lead + (6,)}")
    if steps > 0 and batch > 0:
        nb = (steps + batch - 1) // batch
        if out.batch_sums is None:
            raise ValueError("batch > 0 needs batch_sums")
        need("batch_sums", out.batch_sums, torch.int32,
             lambda s: len(s) == len(lead) + 2 and s[:-2] == lead and rows_ok(s[-2]) and s[-1] == nb,
             f"{lead} + (n_chains={n_chains}, {nb})")
    if steps > 0 and emit_bits:
        rw = bits_row_words or (steps + 31) // 32
        if out.bits is None:
            raise ValueError("emit_bits needs bits")
        if rw < (bits_offset + steps + 31) // 32:
            raise ValueError("bits_row_words too small for bits_offset + steps")
        need("bits", out.bits, torch.int32,
             lambda s: len(s) == len(lead) + 2 and s[:-2] == lead and rows_ok(s[-2]) and s[-1] == rw,
             f"{lead} + (n_chains={n_chains}, {rw})")
    if out.workspace is not None:
        need("workspace", out.workspace, torch.uint8, lambda s: len(s) == 1, "(bytes,)")
        if out.workspace.numel() < pbn_simulate_workspace_size(model, n_chains, n_props):
            raise ValueError("workspace smaller than pbn_simulate_workspace_size()")


def _pred(pred):
    if pred is None or len(pred.nodes) == 0:
        return L.pbn_predicate(0, None, None), None
    nodes = np.ascontiguousarray(pred.nodes, np.uint16)
    vals = np.ascontiguousarray(pred.values, np.uint8)
    return L.pbn_predicate(len(nodes), L._ptr(nodes, C.c_uint16), L._ptr(vals, C.c_uint8)), (nodes, vals)


def _stream_handle(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def pbn_simulate(model: Model, out: SimOutputs, *, n_chains: int, steps: int, chain_base: int = 0,
                 step0: int = 0, burn_in: int = 0, batch: int = 0, seed: int = 0, pred=None,
                 init: bool = False, emit_bits: bool = False, bits_offset: int = 0,
                 bits_row_words: int = 0, groups_per_cta: int = 0, warps_per_group: int = 0,
                 schedule: int = 0, chunk_steps: int = 0, stream=None, props=None,
                 cluster_size: int = 0, layout: int = 0, chains_per_cluster: int = 0) -> None:
    """props: a list of q >= 1 predicates evaluated on the same trajectories
    (multi-property reuse); `pred` is then ignored.  layout:
    PBN_LAYOUT_* (0 auto, 1 chains over lanes, 2 nodes over lanes)."""
    cp, _keep = _pred(pred)
    keep_props = None
    n_props, props_ptr = 0, None
    if props:
        items = [_pred(p) for p in props]
        arr = (L.pbn_predicate * len(items))(*[it[0] for it in items])
        keep_props = (arr, [it[1] for it in items])
        n_props, props_ptr = len(items), C.cast(arr, C.c_void_p)
    a = L.pbn_sim_args(n_chains=n_chains, chain_base=chain_base, step0=step0, burn_in=burn_in,
                       steps=steps, batch=batch, seed=seed, pred=cp, init=int(bool(init)),
                       emit_bits=int(bool(emit_bits)), bits_offset=bits_offset,
                       bits_row_words=bits_row_words, groups_per_cta=groups_per_cta,
                       warps_per_group=warps_per_group, schedule=schedule, chunk_steps=chunk_steps,
                       n_props=n_props, props=props_ptr, cluster_size=cluster_size, layout=layout,
                       chains_per_cluster=chains_per_cluster)
    _check_outputs(model, out, n_chains=n_chains, steps=steps, batch=batch, emit_bits=emit_bits,
                   bits_offset=bits_offset, bits_row_words=bits_row_words, n_props=n_props)
    if out.workspace is not None:
        a.workspace = C.c_void_p(out.workspace.data_ptr())
        a.workspace_bytes = out.workspace.numel()
    o = out.c_struct()
    check(lib().pbn_simulate(model.handle, C.byref(a), C.byref(o), _stream_handle(stream)))
    del keep_props  # the predicate arrays are read synchronously by the call above


def pbn_recount(bits, n_chains: int, row_words: int, start: int, length: int, batch: int = 0,
                c1=None, n01=None, n10=None, first_last=None, batch_sums=None, totals=None,
                stream=None) -> None:
    def p(t):
        return C.c_void_p(t.data_ptr()) if t is not None else None
    check(lib().pbn_recount(p(bits), n_chains, row_words, start, length, batch, p(c1), p(n01), p(n10),
                            p(first_last), p(batch_sums), p(totals), _stream_handle(stream)))


def pbn_gelman_rubin(S1: int, S2: int, omega: int, psi: int):
    """Returns (status, rhat, B, W, sigma2)."""
    r, B, W, s2 = C.c_double(), C.c_double(), C.c_double(), C.c_double()
    st = lib().pbn_gelman_rubin(int(S1), int(S2), int(omega), int(psi), C.byref(r), C.byref(B),
                                C.byref(W), C.byref(s2))
    return st, r.value, B.value, W.value, s2.value


def pbn_two_state(n01: int, n0from: int, n10: int, n1from: int, r: float, s: float, eps: float):
    res = L.pbn_two_state_result()
    st = lib().pbn_two_state(int(n01), int(n0from), int(n10), int(n1from), float(r), float(s),
                             float(eps), C.byref(res))
    return st, res


def pbn_inv_norm_cdf(q: float) -> float:
    return lib().pbn_inv_norm_cdf(float(q))


def pbn_t_quantile(q: float, df: float) -> float:
    return lib().pbn_t_quantile(float(q), float(df))


def pbn_skart_ci_from_batches(batch_sums: np.ndarray, kappa: int, alpha_conf: float):
    """batch_sums: host uint32 [omega x per_chain] (chain-major)."""
    bs = np.ascontiguousarray(batch_sums, dtype=np.uint32)
    omega, per = bs.shape
    res = L.pbn_skart_ci()
    st = lib().pbn_skart_ci_from_batches(bs.ctypes.data_as(C.c_void_p), omega, per, int(kappa),
                                         float(alpha_conf), C.byref(res))
    return st, res


def pbn_skart(bits, omega: int, row_words: int, start: int, available: int, h_star: float, alpha_conf: float,
              stream=None):
    """Skart sizing over device bitstreams (include/pbnsim.h pbn_skart).
    Returns (status, pbn_skart_result): PBN_OK with the CI, or
    PBN_E_NOT_CONVERGED with need_per_chain = samples per chain to simulate
    before calling again."""
    res = L.pbn_skart_result()
    st = lib().pbn_skart(C.c_void_p(bits.data_ptr()), int(omega), int(row_words), int(start), int(available),
                         float(h_star), float(alpha_conf), C.byref(res), _stream_handle(stream))
    return st, res


def pbn_run(model: Model, *, method: int = 0, omega: int, psi0: int, rhat_threshold: float = 1.1,
            r: float = 0.01, s: float = 0.95, eps: float = 1e-10, h_star: float = 1e-3,
            alpha_conf: float = 0.05, seed: int = 0, pred=None, max_steps: int = 1 << 26,
            stream=None):
    cp, _keep = _pred(pred)
    a = L.pbn_run_args(method=method, omega=omega, psi0=psi0, rhat_threshold=rhat_threshold, r=r, s=s,
                       eps=eps, h_star=h_star, alpha_conf=alpha_conf, seed=seed, pred=cp,
                       max_steps=max_steps)
    res = L.pbn_run_result()
    err = C.create_string_buffer(512)
    st = lib().pbn_run(model.handle, C.byref(a), C.byref(res), _stream_handle(stream), err, 512)
    return st, res, err.value.decode(errors="replace")


def pbn_run_multi(model: Model, props, *, omega: int, psi0: int, rhat_threshold: float = 1.1,
                  r: float = 0.01, s: float = 0.95, eps: float = 1e-10, seed: int = 0,
                  max_steps: int = 1 << 26, stream=None):
    """Algorithm 3 + Algorithm 4 for several properties on shared samples
    (P:507-526).  Returns (status, run_result, [per-property results], err)."""
    items = [_pred(p) for p in props]
    arr = (L.pbn_predicate * len(items))(*[it[0] for it in items])
    a = L.pbn_run_args(method=0, omega=omega, psi0=psi0, rhat_threshold=rhat_threshold, r=r, s=s,
                       eps=eps, seed=seed, max_steps=max_steps)
    res = L.pbn_run_result()
    per = (L.pbn_prop_result * len(items))()
    err = C.create_string_buffer(512)
    st = lib().pbn_run_multi(model.handle, C.byref(a), C.cast(arr, C.c_void_p), len(items), C.byref(res),
                             C.cast(per, C.c_void_p), _stream_handle(stream), err, 512)
    del items
    return st, res, list(per), err.value.decode(errors="replace")
