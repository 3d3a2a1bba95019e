"""K1 direct on C3 (4096 lines x 4096, fp64) for ncu: 2 launches."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import api  # noqa: E402

n = 4096
dev = api.Device(0)
K = dev.build_kernel(n, 0.01, 0.0)
u = torch.from_numpy(api.gen_c3_lines(0, 4096, n)).cuda()
o = torch.empty_like(u)
dk = torch.from_numpy(K.window).cuda()
df = torch.full((4096,), K.first, dtype=torch.int64, device="cuda")
for _ in range(2):
    dev.direct_f64(u, o, dk, df)
torch.cuda.synchronize()
print("done")
