"""C4 split step timing, K2L (whole-line kernel, columns in place) vs the tiled fused path,
and a 20-step trajectory comparison of the two (bit-exact) plus K1.
usage: python scripts/time_c4.py [--steps K]"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
import os  # noqa: E402

from paper_1210_4090_b200 import _capi, api  # noqa: E402

if os.environ.get("LOB_LIB"):
    _capi.LIB_PATH = os.path.abspath(os.environ["LOB_LIB"])

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--mode", type=int, default=-1, help="time this fast_line mode only (no checks)")
ap.add_argument("--time", type=int, default=-1, help="time this mode (and check it == K1 after 20 steps)")
a = ap.parse_args()
n, tau = 2048, 0.01
dev = api.Device(0)
am = torch.from_numpy(api.gen_cos(n)).cuda()
u0 = torch.from_numpy(api.gen_c4_u0(n)).cuda()
ws = torch.empty(2 * dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")


def run(line, engine, k0, k, u):
    dev.set_fast_line(line)
    o, t = torch.empty_like(u), torch.empty_like(u)
    u = u.clone()
    for i in range(k0, k0 + k):
        dev.split_step_2d(u, o, t, tau, 0.3, -0.7, a1=am, a2=am, b=api.c4_time_term(i * tau + tau), engine=engine,
                          workspace=ws)
        u, o = o, u
    return u


res = {}
if a.time >= 0:
    ok = bool(torch.equal(run(a.time, api.ENGINE_FAST, 0, 20, u0), run(a.time, api.ENGINE_DIRECT, 0, 20, u0)))
    u = run(a.time, api.ENGINE_FAST, 0, 5, u0)
    torch.cuda.synchronize()
    best = []
    for r in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        u = run(a.time, api.ENGINE_FAST, 5, a.steps, u)
        e1.record()
        torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1) / a.steps)
    print(json.dumps({"mode": a.time, "lib": os.environ.get("LOB_LIB", "default"), "equal_k1": ok, "ms": sorted(best)}))
    sys.exit(0)
if a.mode >= 0:
    u = run(a.mode, api.ENGINE_FAST, 0, a.steps, u0)
    torch.cuda.synchronize()
    print("done")
    sys.exit(0)
ref = run(True, api.ENGINE_DIRECT, 0, 20, u0)
for line in (5, 2, 3, 0):
    got = run(line, api.ENGINE_FAST, 0, 20, u0)
    torch.cuda.synchronize()
    res[f"line={line} == K1 after 20 steps"] = bool(torch.equal(got, ref))
for line in (5, 2, 3, 0):
    u = run(line, api.ENGINE_FAST, 0, 5, u0)
    torch.cuda.synchronize()
    best = []
    for r in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        u = run(line, api.ENGINE_FAST, 5, a.steps, u)
        e1.record()
        torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1) / a.steps)
    res[f"line={line} ms/step"] = sorted(best)
print(json.dumps(res))
