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


def _slab_worker(rank, world, port, q, n, engine, steps):
    """One rank of the row-partitioned split step on the shared GPU; the all-to-all exchange is
    host-staged over gloo (the ranks' kernels never wait on one another)."""
    import os
    import sys

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1210_4090_b200 import api
    from paper_1210_4090_b200.dist import split_step_2d_dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = api.Device(0)
    tau, d1, d2 = 0.01, 0.3, -0.7
    u0 = api.gen_c4_u0(n)
    a = api.gen_cos(n)
    b = n // world
    v = torch.from_numpy(np.ascontiguousarray(u0[rank * b:(rank + 1) * b])).cuda()
    wss = {}
    for step in range(steps):
        v = split_step_2d_dist(dev, v, tau, d1, d2, a1=a, a2=a, b=api.c4_time_term((step + 1) * tau),
                               engine=engine, workspaces=wss, host_staged=True)
    torch.cuda.synchronize()
    q.put((rank, v.cpu().numpy()))
    dist.destroy_process_group()
    dev.close()


@pytest.mark.parametrize("engine", [api.ENGINE_FAST, api.ENGINE_DIRECT])
def test_dist_split_step_two_ranks_equals_single_gpu(dev, engine):
    """world_size 2: two processes, each its row slab on the one GPU, the two all-to-all
    transposes per step host-staged over gloo (pack / unpack by the library's kernels); after
    3 steps the stacked slabs == the single-GPU lob_split_step_2d_f64 chain (C4's kinetics and
    potential, n = 256)."""
    import torch
    import torch.multiprocessing as mp

    n, steps, world = 256, 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29611 + engine
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q, n, engine, steps)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, slab = q.get(timeout=300)
        res[r] = slab
    for p in procs:
        p.join(timeout=60)
    got = np.concatenate([res[r] for r in range(world)])
    tau = 0.01
    u = torch.from_numpy(api.gen_c4_u0(n)).cuda()
    out, tmp = torch.empty_like(u), torch.empty_like(u)
    a = torch.from_numpy(api.gen_cos(n)).cuda()
    ws = torch.empty(2 * dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
    for step in range(steps):
        dev.split_step_2d(u, out, tmp, tau, 0.3, -0.7, a1=a, a2=a, b=api.c4_time_term((step + 1) * tau),
                          engine=engine, workspace=ws)
        u, out = out, u
    torch.cuda.synchronize()
    assert np.array_equal(got, u.cpu().numpy())


@pytest.mark.parametrize("world", [1, 2, 4])
def test_slab_push_writes_every_peer_block(dev, world):
    """lob_slab_push_f64's index map for several ranks on the one GPU: each rank's call (run one
    after another, so no kernel waits on another) writes its blocks of X^T into all receive slabs
    (here plain local buffers standing in for the peers' symmetric-memory slabs); after every rank
    has pushed, slab q == rows [q b, (q+1) b) of X^T."""
    import torch

    from paper_1210_4090_b200 import _capi
    from paper_1210_4090_b200.api import _ptr

    n = 256
    b = n // world
    if b % 64:
        pytest.skip("b % 64")
    rng = np.random.default_rng(world)
    X = rng.standard_normal((n, n))
    dX = torch.from_numpy(X).cuda()
    slabs = [torch.full((b, n), np.nan, dtype=torch.float64, device="cuda") for _ in range(world)]
    ptrs = np.array([s.data_ptr() for s in slabs], dtype=np.uint64)
    for r in range(world):
        x = dX[r * b:(r + 1) * b].contiguous()
        st = dev.lib.lob_slab_push_f64(dev.ctx, _ptr(x), b, world, r, ptrs.ctypes.data, None)
        _capi.check(st, dev.ctx, "lob_slab_push_f64")
        torch.cuda.synchronize()
    XT = X.T
    for q in range(world):
        assert np.array_equal(slabs[q].cpu().numpy(), XT[q * b:(q + 1) * b])


def _p2p_worker(port, q, n, steps):
    """World size 1 with a real process group (NCCL) and CUDA symmetric memory: the split step
    through P2PExchange."""
    import os
    import sys

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1210_4090_b200 import api
    from paper_1210_4090_b200.dist import P2PExchange, split_step_2d_dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    dev = api.Device(0)
    tau, d1, d2 = 0.01, 0.3, -0.7
    u0 = api.gen_c4_u0(n)
    a = api.gen_cos(n)
    ex = P2PExchange(dev, n, n)
    v = torch.from_numpy(np.ascontiguousarray(u0)).cuda()
    u = v.clone()
    out, tmp = torch.empty_like(u), torch.empty_like(u)
    da = torch.from_numpy(a).cuda()
    wss = {}
    ok = True
    for step in range(steps):
        bb = api.c4_time_term((step + 1) * tau)
        v = split_step_2d_dist(dev, v, tau, d1, d2, a1=a, a2=a, b=bb, engine=api.ENGINE_FAST, workspaces=wss, p2p=ex)
        v = v.clone()
        dev.split_step_2d(u, out, tmp, tau, d1, d2, a1=da, a2=da, b=bb, engine=api.ENGINE_FAST)
        u, out = out, u
        torch.cuda.synchronize()
        ok = ok and bool(torch.equal(u, v))
    q.put(ok)
    dist.destroy_process_group()
    dev.close()


def test_dist_split_step_p2p_exchange_world1():
    import multiprocessing as mp
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_p2p_worker, args=(port, q, 256, 5))
    p.start()
    ok = q.get(timeout=300)
    p.join(timeout=60)
    assert ok
