"""Times the weak-KAM device kernels (tropical GEMM, Karp, period matrix) with CUDA events."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import _capi, api  # noqa: E402
import os  # noqa: E402

if os.environ.get("LOB_LIB"):
    _capi.LIB_PATH = os.path.abspath(os.environ["LOB_LIB"])

dev = api.Device(0)
fp = dev.bench_fp64()
rng = np.random.default_rng(0)
for m in (128, 256, 512, 1024):
    A = torch.from_numpy(rng.uniform(-1, 1, (m, m))).cuda()
    B = torch.from_numpy(rng.uniform(-1, 1, (m, m))).cuda()
    C = torch.empty_like(A)
    dev.minplus_gemm(A, B, C)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        dev.minplus_gemm(A, B, C)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 20 * 1e-3
    print(f"gemm n={m}: {t*1e6:.1f} us, {m**3/t/1e12:.2f} T cand/s, {m**3/t/fp['minplus_cand_per_s']:.2%} of ceiling")
for m in (128, 512, 600):
    A = torch.from_numpy(rng.uniform(-1, 1, (m, m))).cuda()
    dev.eigenvalue_karp(A)
    for r in range(3):
        l0 = dev.launches
        t0 = time.perf_counter()
        dev.eigenvalue_karp(A)
        print(f"karp n={m}: {(time.perf_counter()-t0)*1e3:.2f} ms, launches {dev.launches - l0}")
