import sys
sys.path.insert(0, ".")
import numpy as np
from tests import _oracle
from tests import test_edge_cases_gpu as T
from paper_1210_4090_b200 import api
dev = api.Device(0); orc = _oracle.oracle()
bad = 0
for seed in range(12, 260):
    try:
        T.test_seeded_differential_sweep_of_engines.__wrapped__(dev, orc, seed) if hasattr(T.test_seeded_differential_sweep_of_engines, "__wrapped__") else T.test_seeded_differential_sweep_of_engines(dev, orc, seed)
    except AssertionError as e:
        bad += 1
        print("FAIL", seed, str(e)[:200], flush=True)
print("done, failures:", bad)
