"""The row-sharded split step (paper_1210_4090_b200/dist.py) through the CUDA kernels.
One GPU is available here, so this runs world_size 1 (the exchange degenerates to a local
transpose); the exchange itself is covered with world_size 2 and 4 over gloo on CPU
(tests/test_dist_cpu.py).  The slab result must equal lob_split_step_2d_f64 bit for bit."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api
from paper_1210_4090_b200.dist import split_step_2d_dist

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("engine", [api.ENGINE_DIRECT, api.ENGINE_FAST])
@pytest.mark.parametrize("n", [64, 256])
def test_dist_split_step_equals_single_gpu(dev, engine, n):
    import torch

    tau, d1, d2 = (0.05 if n < 128 else 0.01), 0.3, -0.7
    x = np.arange(n) / n
    u0 = np.sin(2 * np.pi * x)[:, None] + np.cos(2 * np.pi * x)[None, :]
    a1 = np.cos(2 * np.pi * x)
    a2 = np.cos(2 * np.pi * x)
    u = torch.from_numpy(np.ascontiguousarray(u0)).cuda()
    v = u.clone()
    out, tmp = torch.empty_like(u), torch.empty_like(u)
    ws = torch.empty(dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
    wss = {}
    da1, da2 = torch.from_numpy(a1).cuda(), torch.from_numpy(a2).cuda()
    for step in range(5):
        b = 0.2 * np.sin(2 * np.pi * (step + 1) * tau)
        dev.split_step_2d(u, out, tmp, tau, d1, d2, a1=da1, a2=da2, b=b, engine=engine, workspace=ws)
        u, out = out, u
        v = split_step_2d_dist(dev, v, tau, d1, d2, a1=a1, a2=a2, b=b, engine=engine, workspaces=wss)
        torch.cuda.synchronize()
        assert torch.equal(u, v), step
