"""ncu driver for the widened rows: tropical GEMM (n = 512 product), Karp (n = 512 cluster
kernel), the relaxed engine (eta = 1e-4, 64 C1-shaped lines) and the semi-discrete step
(64 C1 lines, q = 4).  One call of each, after a warm-up call."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import api  # noqa: E402

dev = api.Device(0)
rng = np.random.default_rng(0)
m = 512
A = torch.from_numpy(rng.uniform(-1, 1, (m, m))).cuda()
B = torch.from_numpy(rng.uniform(-1, 1, (m, m))).cuda()
C = torch.empty_like(A)
for _ in range(2):
    dev.minplus_gemm(A, B, C)
    dev.eigenvalue_karp(A)
n, tau = 1024, 0.05
ks = [dev.build_kernel(n, tau, 0.5)] * 64
kt = torch.from_numpy(ks[0].window).cuda()
fr = torch.full((64,), ks[0].first, dtype=torch.int64, device="cuda")
u = torch.from_numpy(np.tile(api.gen_sin(n), (64, 1))).cuda()
u += torch.from_numpy(rng.uniform(-1e-3, 1e-3, (64, n))).cuda()
o = torch.empty_like(u)
for _ in range(2):
    dev.relaxed_f64(u, o, kt, fr, 1e-4)
    dev.step_semidiscrete(u, o, kt, ks[0].first, 0.0, tau, api.potential_cosine(0.0, -1.0, 1), 4)
torch.cuda.synchronize()
print("done")
