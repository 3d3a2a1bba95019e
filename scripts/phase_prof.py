"""Per-phase cycle split of the fast kernel (needs lib/liblaxol_b200_prof.so,
a -DLOB_PHASE_PROF build).  Cycles are thread 0's, summed over tiles, per update."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1210_4090_b200 import _capi
_capi.LIB_PATH = _capi.LIB_PATH.replace("liblaxol_b200.so", "liblaxol_b200_prof.so")
_capi.load(_capi.LIB_PATH)
from paper_1210_4090_b200 import api  # noqa: E402
n, tau, L = 65536, 0.02, 256
dev = api.Device(0)
dr = torch.from_numpy(api.gen_c2_drifts(256)).cuda()
tv = torch.from_numpy(api.tau_v(api.gen_potential(2, n), tau)).cuda()
x = torch.zeros((L, n), dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
ws = torch.empty(dev.fast_workspace_bytes(L, n), dtype=torch.uint8, device="cuda")
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 300):
    dev.fast_f64(x, y, dr, tau, tv=tv, workspace=ws, flags=api.FAST_STATS_VALID if i else 0); x, y = y, x
ws2 = torch.empty_like(ws)
dev.fast_f64(x, y, dr, tau, tv=tv, workspace=ws2, flags=0)
for i in range(5):
    x, y = y, x
    dev.fast_f64(x, y, dr, tau, tv=tv, workspace=ws2, flags=api.FAST_STATS_VALID)
c = dev.fast_counters(ws2, L, n)
upd = 6 * L * n
print({k: round(v / upd, 3) for k, v in c.items() if k.startswith("cyc") or k in ("sources", "inline_candidates")})
print("mean d-range per tile", c["r6"] / c["tiles"], "max", c["r7"])
