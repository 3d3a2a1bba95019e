"""Multi-GPU 2-D dimension splitting (SURVEY.md §8(e), config C4 sharded by rows).

One process per GPU; the n x n state is partitioned into equal row slabs
(rank r holds rows [r*b, (r+1)*b), b = n / world).  The reference's split step
(proj/src/splitting.cpp:37-99) sweeps axis 0 (columns: whole columns are
needed, the window spans two periods), then axis 1 (rows: local), then
subtracts tau*V once.  Per step:

    slab of U  --all-to-all transpose-->  slab of U^T  --K1/K2 row sweep (kernel 1)-->
    --all-to-all transpose back-->  slab  --K1/K2 row sweep (kernel 2)-->  - tau*V (row slab)

i.e. two exchanges of the whole tensor per step, each carrying (world-1)/world of the state:
``torch.distributed.all_to_all_single`` (NCCL) between library pack / unpack kernels, or — with a
``P2PExchange`` — one kernel per exchange that writes the transposed blocks straight into the
peers' symmetric-memory slabs over NVLink, followed by a symmetric-memory barrier;
the sweeps and the potential are the same device kernels as the single-GPU
``lob_split_step_2d_f64``, with the same IEEE operations, so every rank's slab equals the
corresponding rows of the single-GPU step bit for bit.

The exchange (``transpose_slabs``) is pure data movement; it is tested with
world_size 2 over gloo on CPU (tests/test_dist_cpu.py) and composed with the CUDA
kernels in ``split_step_2d_dist``.
"""
from __future__ import annotations

import numpy as np

from . import _capi
from .api import ENGINE_DIRECT, ENGINE_FAST, Device, InvalidInput, _ptr, _stream_ptr


def _world(group):
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def transpose_slabs(x, group=None, dev: Device | None = None, host_staged: bool = False):
    """x: this rank's row slab (b x n, contiguous) of a row-partitioned n x n matrix X
    (b = n / world).  Returns this rank's row slab of X^T:
    y[c][p*b + i] = X[p*b + i][r*b + c].

    CUDA tensors with `dev`: the send buffer is packed and the receive buffer unpacked by the
    library's kernels (lob_slab_pack_f64 / lob_slab_unpack_f64: one coalesced pass each) and
    the exchange is NCCL's all_to_all_single over NVLink/NVSwitch; host_staged=True moves the
    packed blocks through host memory instead (a gloo group: the multi-process test on one GPU)."""
    import torch
    import torch.distributed as dist

    world, rank = _world(group)
    b, n = x.shape
    if b * world != n:
        raise InvalidInput("transpose_slabs: the row slabs must partition the square evenly")
    on_dev = dev is not None and x.is_cuda
    if on_dev:
        send = torch.empty_like(x)
        _capi.check(dev.lib.lob_slab_pack_f64(dev.ctx, _ptr(x), b, world, _ptr(send), _stream_ptr(None)), dev.ctx,
                    "lob_slab_pack_f64")
        if world == 1:
            return send.view(b, n)
    else:
        if world == 1:
            return x.t().contiguous()
        # block q of the send buffer = X[rank rows][q cols]^T : send[q][c][i] = x[i][q*b + c]
        send = x.view(b, world, b).permute(1, 2, 0).contiguous()
    if host_staged:
        if on_dev:
            torch.cuda.synchronize()
        hs = send.cpu()
        hr = torch.empty_like(hs)
        dist.all_to_all_single(hr, hs, group=group)
        recv = hr.to(x.device)
    else:
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=group)
    # recv[p][c][i] = X[p*b + i][rank*b + c]  ->  y[c][p*b + i]
    if on_dev:
        y = torch.empty_like(x)
        _capi.check(dev.lib.lob_slab_unpack_f64(dev.ctx, _ptr(recv), b, world, _ptr(y), _stream_ptr(None)), dev.ctx,
                    "lob_slab_unpack_f64")
        return y
    return recv.view(world, b, b).permute(1, 0, 2).reshape(b, n).contiguous()


class P2PExchange:
    """The row-slab transpose of the split step over NVLink peer memory: two receive slabs in
    CUDA symmetric memory (torch.distributed._symmetric_memory; one per exchange of a step, so a
    fast rank's next push never lands in a slab a slow rank still reads), and per exchange ONE
    kernel (lob_slab_push_f64) that writes this rank's blocks of X^T straight into every peer's
    slab, then the symmetric-memory barrier on the stream — no NCCL call, no pack / unpack pass.
    Requires an initialised process group with CUDA devices and b % 64 == 0."""

    def __init__(self, dev: Device, b: int, n: int, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        if b * max(1, _world(group)[0]) != n or b % 64:
            raise InvalidInput("P2PExchange: rows per rank must be n / world and a multiple of 64")
        self.dev, self.b, self.n = dev, b, n
        self.world, self.rank = _world(group)
        gname = (group or dist.group.WORLD).group_name
        self.slabs = [symm_mem.empty((b, n), dtype=torch.float64, device="cuda") for _ in range(2)]
        self.handles = [symm_mem.rendezvous(t, gname) for t in self.slabs]
        self.peers = [np.array(h.buffer_ptrs, dtype=np.uint64) for h in self.handles]
        self.k = 0

    def transpose(self, x):
        """x: this rank's row slab (b x n, contiguous CUDA) of X; returns this rank's row slab of
        X^T (a symmetric-memory slab, valid until the next-but-one call)."""
        k = self.k
        self.k ^= 1
        st = self.dev.lib.lob_slab_push_f64(self.dev.ctx, _ptr(x), self.b, self.world, self.rank,
                                            self.peers[k].ctypes.data, _stream_ptr(None))
        _capi.check(st, self.dev.ctx, "lob_slab_push_f64")
        self.handles[k].barrier(channel=k)
        return self.slabs[k]


def split_step_2d_dist(dev: Device, u_slab, tau: float, drift1: float, drift2: float, a1=None, a2=None,
                       b: float = 0.0, engine: int = ENGINE_DIRECT, group=None, workspaces=None,
                       host_staged: bool = False, p2p: "P2PExchange | None" = None):
    """One split step of the row-partitioned periodic n x n tensor (this rank's slab,
    rows [r*b, (r+1)*b) as a torch CUDA tensor).  a1 (length n, the x1 factor of the whole
    grid) and a2 (length n) describe V = a1(x1) a2(x2) + b at the step's sampling time,
    like lob_split_step_2d_f64.  Returns the new slab."""
    import torch

    world, rank = _world(group)
    bl, n = u_slab.shape
    if bl * world != n:
        raise InvalidInput("split_step_2d_dist: rows per rank must be n / world")
    if engine not in (ENGINE_DIRECT, ENGINE_FAST):
        raise InvalidInput("split_step_2d_dist: engine must be ENGINE_DIRECT or ENGINE_FAST")

    cache = workspaces if workspaces is not None else {}

    def cached(key, make):
        v = cache.get(key)
        if v is None:
            v = cache[key] = make()
        return v

    def sweep(src, drift, key):
        # two output buffers per axis alternate, so the slab returned by the previous call survives
        flip = cache.get(key + "/flip", 0)
        cache[key + "/flip"] = flip ^ 1
        out = cached(f"{key}/out{flip}", lambda: torch.empty_like(src))
        if engine == ENGINE_FAST:
            ws = cached(key, lambda: torch.empty(dev.fast_workspace_bytes(bl, n), dtype=torch.uint8,
                                                 device=src.device))
            d = cached(f"{key}/drift{drift!r}", lambda: torch.full((bl,), drift, dtype=torch.float64,
                                                                     device=src.device))
            dev.fast_f64(src, out, d, tau, workspace=ws)
        else:
            k = dev.build_kernel(n, tau, drift)
            kt = torch.from_numpy(k.window).to(src.device)
            fr = torch.full((bl,), k.first, dtype=torch.int64, device=src.device)
            dev.direct_f64(src, out, kt, fr)
        return out

    def exchange(x):
        return p2p.transpose(x) if p2p is not None else transpose_slabs(x, group, dev, host_staged)

    t = exchange(u_slab)                  # slab of U^T: columns of U as rows
    t = sweep(t, drift1, "axis0")         # axis 0 (kernel 1)
    v = exchange(t)                       # back to rows
    w = sweep(v, drift2, "axis1")               # axis 1 (kernel 2)
    if a1 is not None:
        a1d = cached("a1/" + str(hash(np.asarray(a1).tobytes())), lambda: torch.as_tensor(np.ascontiguousarray(a1[rank * bl:(rank + 1) * bl]),
                                                             device=w.device))
        a2d = cached("a2/" + str(hash(np.asarray(a2).tobytes())), lambda: torch.as_tensor(np.ascontiguousarray(a2), device=w.device))
        st = dev.lib.lob_potential2d_rows_f64(dev.ctx, _ptr(w), bl, n, _ptr(a1d), _ptr(a2d), float(b), float(tau),
                                              _stream_ptr(None))
        _capi.check(st, dev.ctx, "lob_potential2d_rows_f64")
    return w
