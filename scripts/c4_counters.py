"""Walk counters of one C4 axis-0 sweep (K2L and tiled) after a few split steps."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import api  # noqa: E402

n, tau = 2048, 0.01
dev = api.Device(0)
am = torch.from_numpy(api.gen_cos(n)).cuda()
u = torch.from_numpy(api.gen_c4_u0(n)).cuda()
o, t = torch.empty_like(u), torch.empty_like(u)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    dev.split_step_2d(u, o, t, tau, 0.3, -0.7, a1=am, a2=am, b=api.c4_time_term(i * tau + tau), engine=api.ENGINE_FAST)
    u, o = o, u
ut = u.t().contiguous()
for mode in (2, 0):
    dev.set_fast_line(mode)
    ws = torch.empty(dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(ut)
    dev.fast_f64(ut, out, torch.full((n,), 0.3, dtype=torch.float64, device="cuda"), tau, workspace=ws)
    torch.cuda.synchronize()
    c = dev.fast_counters(ws, n, n)
    print(json.dumps({"mode": mode, **{k: v / (n * n) for k, v in c.items() if k in ("sources", "queued_candidates", "queued_intervals")}, "tiles": c["tiles"], "direct": c["direct_tiles_gate"] + c["direct_tiles_heavy"]}))
