"""C3 fast-path driver for ncu (4096 x 4096 random-walk lines, one step)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import api  # noqa: E402

n = 4096
dev = api.Device(0)
u = torch.from_numpy(api.gen_c3_lines(0, 4096, n)).cuda()
o = torch.empty_like(u)
ws = torch.empty(dev.fast_workspace_bytes(4096, n), dtype=torch.uint8, device="cuda")
z = torch.zeros(4096, dtype=torch.float64, device="cuda")
for _ in range(2):
    dev.fast_f64(u, o, z, 0.01, workspace=ws)
torch.cuda.synchronize()
print("done")
