import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests.helpers import gpu_run, oracle_run, pack_states, unpack_states
import paper_1508_07828_b200 as pbn
from workloads import config_model, config_predicate
for key in ("C2", "C5"):
    model, pred = config_model(key), config_predicate(key)
    pm = pbn.pbn_load(model)
    for steps in (0, 1, 2):
        st, I, ws = oracle_run(model, pred, list(range(8)), steps=steps, burn_in=0, seed=5, batch=0)
        g = gpu_run(pm, model, pred, n_chains=8, steps=steps, burn_in=0, seed=5, cluster_size=1, schedule=1)
        gs = unpack_states(g["state"], model.n)
        diff = np.argwhere(gs != st)
        print(key, "steps", steps, "mismatches", len(diff), diff[:6].tolist(), flush=True)
