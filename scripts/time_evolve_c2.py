"""C2 (256 x 65536) through lob_evolve_f64 (the reference's evolve API: per-step drift and block
counts): time per step after 1000 pre-steps (CUDA events)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import api  # noqa: E402

n, L, tau = 65536, 256, 0.02
dev = api.Device(0)
dr = torch.from_numpy(api.gen_c2_drifts(L)).cuda()
tv = torch.from_numpy(api.tau_v(api.gen_potential(2, n), tau)).cuda()
u = torch.zeros((L, n), dtype=torch.float64, device="cuda")
scr = torch.empty_like(u)
ws = torch.empty(dev.fast_workspace_bytes(L, n), dtype=torch.uint8, device="cuda")
dev.evolve(u, scr, dr, tau, 1000, tv=tv, workspace=ws)
steps = 500
sd = torch.empty(steps * L, dtype=torch.float64, device="cuda")
sb = torch.empty(steps * L, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
dev.evolve(u, scr, dr, tau, steps, tv=tv, step_drift=sd, step_blocks=sb, workspace=ws)
e.record()
torch.cuda.synchronize()
print(json.dumps({"evolve_ms_per_step": s.elapsed_time(e) / steps}))
