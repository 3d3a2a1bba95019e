"""Time the C2 fast step (CUDA events) after --pre steps."""
import argparse, sys
import torch
sys.path.insert(0, ".")
from paper_1210_4090_b200 import api  # noqa: E402
ap = argparse.ArgumentParser(); ap.add_argument("--pre", type=int, default=300)
ap.add_argument("--ablate", type=int, default=0); a = ap.parse_args()
import os
n, tau, L = 65536, 0.02, 256
dev = api.Device(0)
dr = torch.from_numpy(api.gen_c2_drifts(256)).cuda()
tv = torch.from_numpy(api.tau_v(api.gen_potential(2, n), tau)).cuda()
x = torch.zeros((L, n), dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
ws = torch.empty(dev.fast_workspace_bytes(L, n), dtype=torch.uint8, device="cuda")
for i in range(a.pre):
    dev.fast_f64(x, y, dr, tau, tv=tv, workspace=ws, flags=api.FAST_STATS_VALID if i else 0); x, y = y, x
torch.cuda.synchronize()
# time the same input repeatedly (stats stay valid: re-run from x each time)
x0 = x.clone(); ws0 = ws.clone()
if a.ablate:
    os.environ["LOB_FAST_ABLATE"] = str(a.ablate)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(20):
    dev.fast_f64(x0, y, dr, tau, tv=tv, workspace=ws, flags=0)
e1.record(); torch.cuda.synchronize()
print("step+stats (flags=0) ms", e0.elapsed_time(e1) / 20)
