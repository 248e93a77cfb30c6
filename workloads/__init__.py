"""Seeded synthetic PBN workloads (inputs only).

This module is the ONE place shared by the CPU oracle (`oracle/`) and the
B200 product path (`paper_1508_07828_b200/`).  It draws random network
structure and run parameters and holds none of the method's arithmetic:
no thresholds, no Philox, no stepping, no statistics.

Generator per PAPER.md §5.1 (node number, min/max predictor
functions per node, min/max parents per function) with the distributions
the paper leaves open fixed by BASELINE.json configs C1-C5 and
SURVEY.md §8(c) Q14 (parents uniform without replacement over all n
nodes, self allowed; Dirichlet(1..1) selection probabilities; Bernoulli
truth-table bits).
"""
from .generate import (  # noqa: F401
    PbnModel,
    Predicate,
    RunConfig,
    CONFIGS,
    random_pbn,
    config_model,
    config_predicate,
    model_from_lists,
)
