"""C2-like K2 step time vs number of lines (tail/wave quantisation probe)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import api  # noqa: E402

n, tau = 65536, 0.02
dev = api.Device(0)
res = {}
for L in [int(x) for x in sys.argv[1:]]:
    dr = torch.from_numpy(api.gen_c2_drifts(256)[[(i % 23) * 11 for i in range(L)]]).cuda()
    tv = torch.from_numpy(api.tau_v(api.gen_potential(2, n), tau)).cuda()
    x = torch.zeros((L, n), dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ws = torch.empty(dev.fast_workspace_bytes(L, n), dtype=torch.uint8, device="cuda")
    bl = torch.empty(L, dtype=torch.int64, device="cuda")
    for i in range(600):
        dev.fast_f64(x, y, dr, tau, tv=tv, blocks=bl, workspace=ws, flags=api.FAST_STATS_VALID if i else 0)
        x, y = y, x
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(50):
        dev.fast_f64(x, y, dr, tau, tv=tv, blocks=bl, workspace=ws, flags=api.FAST_STATS_VALID)
        x, y = y, x
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    res[L] = {"ms": ms, "us_per_line": ms * 1e3 / L, "waves": L * 32 / (148 * 5)}
print(json.dumps(res))
