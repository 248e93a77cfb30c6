import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests.helpers import gpu_run, oracle_run, pack_states
import paper_1508_07828_b200 as pbn
from workloads import config_model, config_predicate
model, pred = config_model("C5"), config_predicate("C5")
pm = pbn.pbn_load(model)
st, I, ws = oracle_run(model, pred, [0, 1, 33], steps=50, burn_in=0, seed=5, batch=0)
packed = pack_states(st)
for W in (8, 16):
    for sched in (1, 2):
        g = gpu_run(pm, model, pred, n_chains=40, steps=50, burn_in=0, seed=5, warps=W, cluster_size=1, schedule=sched)
        ok = [np.array_equal(g["state"][c], packed[k]) for k, c in enumerate([0, 1, 33])]
        print("W", W, "sched", sched, ok, flush=True)
for steps in (1, 2, 3):
    st, I, ws = oracle_run(model, pred, [0], steps=steps, burn_in=0, seed=5, batch=0)
    g = gpu_run(pm, model, pred, n_chains=1, steps=steps, burn_in=0, seed=5, cluster_size=1, schedule=1)
    print("steps", steps, np.array_equal(g["state"][0], pack_states(st)[0]), flush=True)
