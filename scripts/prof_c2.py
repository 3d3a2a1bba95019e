"""C2 fast-path driver for ncu: evolve --pre steps, then --steps more."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import _capi, api  # noqa: E402
import os  # noqa: E402

if os.environ.get("LOB_LIB"):
    _capi.LIB_PATH = os.path.abspath(os.environ["LOB_LIB"])

ap = argparse.ArgumentParser()
ap.add_argument("--pre", type=int, default=300)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--lines", type=int, default=256)
ap.add_argument("--blocks", action="store_true", help="request decompose() block counts")
a = ap.parse_args()
n, tau, L = 65536, 0.02, a.lines
dev = api.Device(0)
dr = torch.from_numpy(api.gen_c2_drifts(256)[:L]).cuda()
tv = torch.from_numpy(api.tau_v(api.gen_potential(2, n), tau)).cuda()
x = torch.zeros((L, n), dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
ws = torch.empty(dev.fast_workspace_bytes(L, n), dtype=torch.uint8, device="cuda")
for i in range(a.pre + a.steps):
    dev.fast_f64(x, y, dr, tau, tv=tv, workspace=ws, flags=api.FAST_STATS_VALID if i else 0)
    x, y = y, x
torch.cuda.synchronize()
print("done", float(x.mean()))
ws2 = torch.empty_like(ws)
bl = torch.empty(L, dtype=torch.int64, device="cuda") if a.blocks else None
dev.fast_f64(x, y, dr, tau, tv=tv, blocks=bl, workspace=ws2, flags=0)
for i in range(5):
    x, y = y, x
    dev.fast_f64(x, y, dr, tau, tv=tv, blocks=bl, workspace=ws2, flags=api.FAST_STATS_VALID)
c = dev.fast_counters(ws2, L, n)
upd = 6 * L * n
print({k: v / upd for k, v in c.items()}, c)
