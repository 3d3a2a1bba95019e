"""Multi-process (world_size 2, gloo, CPU) coverage of bench.py's N>1 path:
rendezvous on 127.0.0.1, barrier, max-over-ranks timing, rank-0-only
output of the reference arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench.barrier(world)
    m = bench.allreduce_max(float(rank + 1) * 1.5, world, device="cpu")
    q.put((rank, m))
    dist.destroy_process_group()


def test_allreduce_max_over_ranks_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29517
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: 3.0, 1: 3.0}


@pytest.mark.slow
def test_bench_reference_arm_two_ranks():
    """torchrun --nproc-per-node 2 bench.py --impl reference: rank 0 alone prints one JSON line."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liblaxol_ref.so")):
        pytest.skip("reference build absent")
    env = dict(os.environ, OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-lines", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "updates/s"


def _transpose_worker(rank, world, port, q, n):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1210_4090_b200.dist import transpose_slabs

    dist.init_process_group("gloo", rank=rank, world_size=world)
    X = np.arange(n * n, dtype=np.float64).reshape(n, n) * 1.5 - 7.0
    b = n // world
    x = torch.from_numpy(X[rank * b:(rank + 1) * b].copy())
    y = transpose_slabs(x)
    z = transpose_slabs(y)  # back
    q.put((rank, y.numpy(), z.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 8), (2, 12), (4, 16)])
def test_all_to_all_transpose_of_row_slabs_gloo(world, n):
    """The C4 multi-GPU exchange (paper_1210_4090_b200/dist.py): every rank's slab of the
    all-to-all transpose is the matching rows of X^T, and transposing twice is the identity."""
    import numpy as np
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29541 + world + n
    procs = [ctx.Process(target=_transpose_worker, args=(r, world, port, q, n)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, y, z = q.get(timeout=180)
        res[r] = (y, z)
    for p in procs:
        p.join(timeout=60)
    X = np.arange(n * n, dtype=np.float64).reshape(n, n) * 1.5 - 7.0
    b = n // world
    for r in range(world):
        assert np.array_equal(res[r][0], X.T[r * b:(r + 1) * b])
        assert np.array_equal(res[r][1], X[r * b:(r + 1) * b])
