"""C4 fused split step: the fast engine's counters of each axis' workspace half after a few steps."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import api  # noqa: E402

n, tau = 2048, 0.01
dev = api.Device(0)
am = torch.from_numpy(api.gen_cos(n)).cuda()
u = torch.from_numpy(api.gen_c4_u0(n)).cuda()
o, t = torch.empty_like(u), torch.empty_like(u)
wsz = dev.fast_workspace_bytes(n, n)
ws = torch.empty(2 * wsz, dtype=torch.uint8, device="cuda")
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    dev.split_step_2d(u, o, t, tau, 0.3, -0.7, a1=am, a2=am, b=api.c4_time_term(i * tau + tau), workspace=ws,
                      engine=api.ENGINE_FAST)
    u, o = o, u
torch.cuda.synchronize()
for h in range(2):
    c = dev.fast_counters(ws[h * wsz:(h + 1) * wsz], n, n)
    upd = max(1, c["tiles"]) * n
    print("axis", h, {k: (v / upd if k in ("sources", "queued_candidates", "queued_intervals", "k_range_sum") else v) for k, v in c.items()})
