"""Quick device timings of K1 (C3) and K2 (C2, C5) + FP64 micro-benchmark."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import api  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


dev = api.Device(0)
res = {"fp64": dev.bench_fp64()}
# K1 C3 fp64
n = 4096
K = dev.build_kernel(n, 0.01, 0.0)
u = torch.from_numpy(api.gen_c3_lines(0, 4096, n)).cuda()
out = torch.empty_like(u)
dk = torch.from_numpy(K.window).cuda()
df = torch.full((4096,), K.first, dtype=torch.int64, device="cuda")
t = timeit(lambda: dev.direct_f64(u, out, dk, df), reps=5, warm=2)
cands = 4096 * 4096 * (2 * n + 1)
res["k1_c3_f64"] = {"s": t, "updates_per_s": 4096 * 4096 / t, "cand_per_s": cands / t}
u32 = u.float()
o32 = torch.empty_like(u32)
dk32 = dk.float()
t = timeit(lambda: dev.direct_f32(u32, o32, dk32, df), reps=5, warm=2)
res["k1_c3_f32"] = {"s": t, "updates_per_s": 4096 * 4096 / t, "cand_per_s": cands / t}
# K2 on C3
ws = torch.empty(dev.fast_workspace_bytes(4096, n), dtype=torch.uint8, device="cuda")
dz = torch.zeros(4096, dtype=torch.float64, device="cuda")
t = timeit(lambda: dev.fast_f64(u, out, dz, 0.01, workspace=ws), reps=10)
res["k2_c3"] = {"s": t, "updates_per_s": 4096 * 4096 / t}
# K2 on C2 (evolved 50 steps from 0)
n = 65536
tau = 0.02
dr = torch.from_numpy(api.gen_c2_drifts(256)).cuda()
tv = torch.from_numpy(api.tau_v(api.gen_potential(2, n), tau)).cuda()
a = torch.zeros((256, n), dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
ws = torch.empty(dev.fast_workspace_bytes(256, n), dtype=torch.uint8, device="cuda")
state = {"a": a, "b": b, "i": 0}


def c2step():
    dev.fast_f64(state["a"], state["b"], dr, tau, tv=tv, workspace=ws,
                 flags=api.FAST_STATS_VALID if state["i"] else 0)
    state["a"], state["b"] = state["b"], state["a"]
    state["i"] += 1


for _ in range(50):
    c2step()
t = timeit(c2step, reps=20)
res["k2_c2"] = {"s": t, "updates_per_s": 256 * n / t, "hbm_frac": 256 * n * 16 / t / 6443.8e9,
                "after_steps": state["i"]}
print(json.dumps(res, indent=1))
