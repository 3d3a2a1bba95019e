import sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1210_4090_b200 import api
from tests import _oracle
from tests.test_weakkam import _device_period_matrix, cos_table
dev = api.Device(0)
ref = _oracle.reference()
for n in (32, 48, 64):
    C = _device_period_matrix(dev, n, 0.125, 0.0, cos_table(n))
    ch = C.cpu().numpy()
    want = ref.karp(ch)[0]
    got = [dev.eigenvalue_karp(C) for _ in range(5)]
    print(n, want, got)
    rng = np.random.default_rng(1)
    m = rng.uniform(-2, 2, (n, n))
    print(" rand", ref.karp(m)[0], [dev.eigenvalue_karp(torch.from_numpy(m).cuda()) for _ in range(3)])
