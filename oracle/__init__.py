"""CPU oracle for the PBN trajectory hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import anything under `oracle/`.  The product
path (`paper_1508_07828_b200`) never imports it and shares no code with it;
only the seeded input generators in `workloads/` serve both.

Modules
  pbn_oracle.c  Philox4x32-10, thresholds, one step, trajectories (plain C)
  sim.py        ctypes marshalling for pbn_oracle.c
  stats.py      per-chain statistics by definition, Gelman & Rubin,
                two-state, Phi^-1, Student-t quantile, Skart (fp64)
  exact.py      exact 2^n transition matrix (two independent builders)
                and stationary distribution (power iteration + LU)
  driver.py     Algorithms 3, 4, 5 of PAPER.md over the oracle simulator

Parity status per function is listed in DESIGN.md §Oracle.  Skart control
flow beyond SPEC.md's declared constants is "parity unpinned" (the paper
defers it to [AJE08]).
"""
