"""Seeded sweep of split_step_nd (periodic ranks 1-3 with every engine, and windowed tensors of
ragged shapes) and of the tropical GEMM / Karp eigenvalue against the reference library.
usage: fuzz_nd.py [seeds]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from tests import _oracle
from paper_1210_4090_b200 import api

dev = api.Device(0)
ref = _oracle.reference()
nseeds = int(sys.argv[1]) if len(sys.argv) > 1 else 60
fails = checks = 0


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def fail(what, seed, **kw):
    global fails
    fails += 1
    print("FAIL", what, seed, kw, flush=True)


for seed in range(nseeds):
    rng = np.random.default_rng(60000 + seed)
    # ---- periodic split_step_nd ----
    rank = int(rng.integers(1, 4))
    n = int(rng.integers(3, {1: 400, 2: 48, 3: 14}[rank]))
    tau = 1.0 / (n * float(rng.uniform(0.05, 0.95)))
    drifts = [float(d) for d in (rng.uniform(-3, 3, rank) if rng.random() < 0.3 else rng.uniform(-1.2, 1.2, rank)) / tau]
    shape = (n,) * rank
    u = rng.uniform(-1, 1, shape) * rng.uniform(0.01, 1)
    for a in range(rank):
        idx = [None] * rank
        idx[a] = slice(None)
        u = u + np.sin(2 * np.pi * (a + 1) * np.arange(n) / n)[tuple(idx)]
    v = rng.uniform(-1, 1, shape)
    try:
        for eng, eta in ((api.ENGINE_DIRECT, 0.0), (api.ENGINE_FAST, 0.0), (api.ENGINE_RELAXED, 1e-5)):
            want = ref.split_step_nd(u, rank, n, tau, drifts, vtab=v, eta=eta)
            for mode in ((2, 0) if eng == api.ENGINE_FAST else (2,)):
                dev.set_fast_line(mode)
                du = t(u.ravel())
                out, tmp = torch.empty_like(du), torch.empty_like(du)
                ks = [dev.build_kernel(n, tau, d) for d in drifts]
                ws = torch.empty(dev.fast_workspace_bytes(n ** (rank - 1), n), dtype=torch.uint8, device="cuda")
                dev.split_step_nd(du, out, tmp, rank, n, tau, kernels=ks, drifts=drifts, tv=t((tau * v).ravel()), eta=eta,
                                  engine=eng, workspace=ws)
                torch.cuda.synchronize()
                checks += 1
                if not np.array_equal(out.cpu().numpy(), want):
                    fail("split_nd", seed, rank=rank, n=n, tau=tau, tp=[d * tau for d in drifts], eng=eng, mode=mode)
        dev.set_fast_line(2)
    except Exception as exc:
        dev.set_fast_line(2)
        fail("split_nd exception", seed, rank=rank, n=n, err=str(exc)[:200])
    # ---- windowed tensors of ragged shapes ----
    try:
        wr = int(rng.integers(1, 4))
        dims = tuple(int(x) for x in rng.integers(2, {1: 200, 2: 40, 3: 12}[wr], wr))
        nsp = int(rng.integers(4, 40))
        tw = 1.0 / (nsp * float(rng.uniform(0.1, 0.9)))
        wd = [float(x) for x in rng.uniform(-1.0, 1.0, wr) / tw]
        org = [float(x) for x in rng.uniform(-1, 1, wr)]
        uw = rng.uniform(-1, 1, dims)
        vw = rng.uniform(-1, 1, dims)
        want, st = ref.split_step_nd_window(uw, nsp, tw, wd, org, vtab=vw)
        du = t(uw.ravel())
        out, tmp = torch.empty_like(du), torch.empty_like(du)
        ks = [dev.build_kernel(nsp, tw, d) for d in wd]
        try:
            dev.split_step_nd_window(du, out, tmp, dims, nsp, tw, ks, tv=t((tw * vw).ravel()))
            torch.cuda.synchronize()
            got_st = 0
        except api.EvaluationError:
            got_st = 2
        checks += 1
        if (st != 0) != (got_st != 0):
            fail("split_nd_window status", seed, dims=dims, n=nsp, st=st, got=got_st)
        elif st == 0 and not np.array_equal(out.cpu().numpy(), want):
            fail("split_nd_window", seed, dims=dims, n=nsp, tau=tw)
    except Exception as exc:
        fail("split_nd_window exception", seed, err=str(exc)[:200])
    # ---- tropical GEMM and Karp ----
    try:
        m = int(rng.integers(1, 70))
        A = rng.uniform(-2, 2, (m, m))
        B = rng.uniform(-2, 2, (m, m))
        if rng.random() < 0.3:
            A[rng.random((m, m)) < 0.2] = np.inf
            B[rng.random((m, m)) < 0.2] = np.inf
        want = ref.minplus_product(A, B)
        want = want[0] if isinstance(want, tuple) else want
        o = torch.empty((m, m), dtype=torch.float64, device="cuda")
        dev.minplus_gemm(t(A), t(B), o)
        torch.cuda.synchronize()
        checks += 1
        if not np.array_equal(o.cpu().numpy(), np.asarray(want).reshape(m, m)):
            fail("gemm", seed, m=m)
    except Exception as exc:
        fail("gemm exception", seed, err=str(exc)[:200])
print("done, checks:", checks, "failures:", fails)
