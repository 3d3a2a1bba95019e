"""C4 split step (2048^2, P=(0.3,-0.7), V=cos cos + 0.2 sin 2 pi t) for ncu: --steps split steps."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import _capi, api  # noqa: E402
import os  # noqa: E402

if os.environ.get("LOB_LIB"):
    _capi.LIB_PATH = os.path.abspath(os.environ["LOB_LIB"])

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--engine", type=int, default=api.ENGINE_FAST)
ap.add_argument("--halves", type=int, default=2, help="workspace halves (2: the fused four-launch step)")
a = ap.parse_args()
n, tau = 2048, 0.01
dev = api.Device(0)
am = torch.from_numpy(api.gen_cos(n)).cuda()
u = torch.from_numpy(api.gen_c4_u0(n)).cuda()
o, t = torch.empty_like(u), torch.empty_like(u)
ws = torch.empty(a.halves * dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
for i in range(a.steps):
    dev.split_step_2d(u, o, t, tau, 0.3, -0.7, a1=am, a2=am, b=api.c4_time_term(i * tau + tau), engine=a.engine,
                      workspace=ws)
    u, o = o, u
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(a.steps, a.steps + 50):
    dev.split_step_2d(u, o, t, tau, 0.3, -0.7, a1=am, a2=am, b=api.c4_time_term(i * tau + tau), engine=a.engine,
                      workspace=ws)
    u, o = o, u
e1.record()
torch.cuda.synchronize()
print("ok", float(u.mean()), "ms/step", e0.elapsed_time(e1) / 50)
