"""Oracle multi-property driver (reading Q13), pinned on CPU:
  - with one property it is exactly the single-property Algorithm 4 driver;
  - the pooled sample is shared: its size is below the sum of the sizes of
    separate single-property runs (the saving the paper reports in Table 2,
    P:797-815: 452.74 vs 1563.05 million), and at least the largest of them
    is not required (only the largest N must be met);
  - every non-degenerate property's N is met by the pooled sample.
"""
import numpy as np

from oracle import driver as odr
from workloads import Predicate, config_model, config_predicate

ARGS = dict(seed=3, omega=8, psi0=300, threshold=1.1, r=0.02, s=0.95, eps=1e-10, max_steps=1 << 22)


def test_single_property_reduces_to_algorithm_4():
    m, p = config_model("C1"), config_predicate("C1")
    a = odr.parallel_two_state(m, p, ARGS["seed"], ARGS["omega"], ARGS["psi0"], ARGS["threshold"], ARGS["r"],
                               ARGS["s"], ARGS["eps"], ARGS["max_steps"])
    b = odr.parallel_two_state_multi(m, [p], ARGS["seed"], ARGS["omega"], ARGS["psi0"], ARGS["threshold"],
                                     ARGS["r"], ARGS["s"], ARGS["eps"], ARGS["max_steps"])
    assert (a.psi, a.extensions, a.sample_size, a.steps_per_chain) == (b.psi, b.extensions, b.sample_size,
                                                                       b.steps_per_chain)
    assert (a.M, a.N) == (b.per_prop[0]["M"], b.per_prop[0]["N"])
    assert a.estimate == b.per_prop[0]["estimate"]


def test_shared_sample_is_smaller_than_separate_runs_and_meets_every_N():
    m = config_model("C1")
    props = [Predicate(np.array([0], np.uint16), np.array([1], np.uint8)),
             Predicate(np.array([1, 2], np.uint16), np.array([1, 0], np.uint8)),
             Predicate(np.array([3, 4, 5], np.uint16), np.array([0, 1, 1], np.uint8))]
    multi = odr.parallel_two_state_multi(m, props, ARGS["seed"], ARGS["omega"], ARGS["psi0"], ARGS["threshold"],
                                         ARGS["r"], ARGS["s"], ARGS["eps"], ARGS["max_steps"])
    singles = [odr.parallel_two_state(m, p, ARGS["seed"], ARGS["omega"], ARGS["psi0"], ARGS["threshold"],
                                      ARGS["r"], ARGS["s"], ARGS["eps"], ARGS["max_steps"]) for p in props]
    assert multi.sample_size < sum(x.sample_size for x in singles)
    for pp in multi.per_prop:
        if not pp["degenerate"]:
            assert pp["N"] <= multi.sample_size
    # the same trajectories: each property's estimate is the mean of its own
    # meta-state sequence, a probability
    assert all(0.0 <= pp["estimate"] <= 1.0 for pp in multi.per_prop)
