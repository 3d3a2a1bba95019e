"""split_step_nd for periodic tensors of rank 1..3 (proj/src/splitting.cpp:37-99) through
lob_split_step_nd_f64 against the reference's own split_step_nd: every engine `==` (the
relaxed engine with eta > 0 reproduces the reference's default-engine approximation), with a
general (non-separable) potential table."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api

pytestmark = pytest.mark.gpu


def _run(dev, u, rank, n, tau, drifts, tv, eta, engine):
    import torch

    du = torch.from_numpy(np.ascontiguousarray(u).ravel()).cuda()
    out, tmp = torch.empty_like(du), torch.empty_like(du)
    ks = [dev.build_kernel(n, tau, d) for d in drifts]
    ws = torch.empty(dev.fast_workspace_bytes(n ** (rank - 1), n), dtype=torch.uint8, device="cuda")
    dtv = None if tv is None else torch.from_numpy(np.ascontiguousarray(tv).ravel()).cuda()
    dev.split_step_nd(du, out, tmp, rank, n, tau, kernels=ks, drifts=drifts, tv=dtv, eta=eta, engine=engine,
                      workspace=ws)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("rank,n,tau", [(1, 64, 0.05), (2, 32, 0.05), (3, 16, 0.1), (3, 24, 0.05)])
@pytest.mark.parametrize("engine", [api.ENGINE_DIRECT, api.ENGINE_FAST, api.ENGINE_RELAXED])
def test_split_nd_equals_reference(dev, ref, rank, n, tau, engine):
    rng = np.random.default_rng(rank * 100 + n)
    shape = (n,) * rank
    x = [np.arange(n) / n] * rank
    grids = np.meshgrid(*x, indexing="ij")
    u = sum(np.sin(2 * np.pi * (a + 1) * g + a) for a, g in enumerate(grids)) + rng.uniform(-1e-3, 1e-3, shape)
    v = np.cos(2 * np.pi * grids[0]) * np.sin(2 * np.pi * grids[-1] + 0.3) + 0.1 * grids[0] * grids[-1]
    drifts = [0.3, -0.7, 0.45][:rank]
    eta = 1e-4 if engine == api.ENGINE_RELAXED else 0.0
    want = ref.split_step_nd(u, rank, n, tau, drifts, vtab=v, eta=eta)
    got = _run(dev, u, rank, n, tau, drifts, tau * v, eta, engine)
    assert np.array_equal(got, want)
    # without the potential
    want0 = ref.split_step_nd(u, rank, n, tau, drifts, eta=eta)
    assert np.array_equal(_run(dev, u, rank, n, tau, drifts, None, eta, engine), want0)


def test_split_nd_rank2_matches_the_2d_entry(dev):
    """rank 2 through lob_split_step_nd_f64 == lob_split_step_2d_f64 with the separable potential"""
    import torch

    n, tau, d1, d2 = 128, 0.02, 0.3, -0.7
    x = np.arange(n) / n
    u = np.sin(2 * np.pi * x)[:, None] + np.cos(2 * np.pi * x)[None, :]
    a1, a2, b = np.cos(2 * np.pi * x), np.cos(2 * np.pi * x), 0.05
    du = torch.from_numpy(u.copy()).cuda()
    out, tmp = torch.empty_like(du), torch.empty_like(du)
    dev.split_step_2d(du, out, tmp, tau, d1, d2, a1=torch.from_numpy(a1).cuda(), a2=torch.from_numpy(a2).cuda(),
                      b=b, engine=api.ENGINE_DIRECT)
    v = a1[:, None] * a2[None, :] + b  # the same two IEEE roundings as the device (product, sum)
    got = _run(dev, u, 2, n, tau, [d1, d2], tau * v, 0.0, api.ENGINE_DIRECT)
    assert np.array_equal(got, out.cpu().numpy().ravel())


@pytest.mark.parametrize("dims,n,tau", [((40,), 16, 0.25), ((20, 30), 16, 0.25), ((12, 16, 10), 8, 0.25)])
def test_split_nd_windowed_equals_reference(dev, ref, dims, n, tau):
    """walls (non-periodic tensors, proj/src/splitting.cpp:66-76 with scheme.cpp:135-144)"""
    import torch

    rng = np.random.default_rng(sum(dims))
    u = rng.uniform(-1, 1, dims)
    origins = [-0.5, 0.25, 0.0][:len(dims)]
    drifts = [0.0, 0.5, -0.25][:len(dims)]
    v = rng.uniform(-1, 1, dims)
    want, st = ref.split_step_nd_window(u, n, tau, drifts, origins, vtab=v)
    assert st == 0
    du = torch.from_numpy(u.ravel().copy()).cuda()
    out, tmp = torch.empty_like(du), torch.empty_like(du)
    ks = [dev.build_kernel(n, tau, d) for d in drifts]
    dev.split_step_nd_window(du, out, tmp, dims, n, tau, ks, tv=torch.from_numpy((tau * v).ravel()).cuda())
    assert np.array_equal(out.cpu().numpy(), want)


def test_split_nd_rank3_with_more_than_65535_lines_per_sweep(dev):
    """A 256^3 tensor has 65536 lines per axis sweep, one more than a grid dimension holds: the
    fast engine (lines folded over two grid dimensions; whole-line and tiled kernels) == the direct
    engine (a flat grid) on every point, with a potential."""
    rank, n, tau = 3, 256, 0.02
    rng = np.random.default_rng(256)
    x = np.arange(n) / n
    g = np.meshgrid(x, x, x, indexing="ij")
    u = np.sin(2 * np.pi * g[0]) + np.cos(4 * np.pi * g[1] + 0.5) * np.sin(2 * np.pi * g[2]) + \
        rng.uniform(-1e-3, 1e-3, (n,) * 3)
    v = np.cos(2 * np.pi * g[0]) * np.cos(2 * np.pi * g[2]) + 0.3 * np.sin(2 * np.pi * g[1])
    drifts = [0.3, -0.7, 0.45]
    want = _run(dev, u, rank, n, tau, drifts, tau * v, 0.0, api.ENGINE_DIRECT)
    for mode in (2, 0):
        dev.set_fast_line(mode)
        try:
            got = _run(dev, u, rank, n, tau, drifts, tau * v, 0.0, api.ENGINE_FAST)
        finally:
            dev.set_fast_line(2)
        assert np.array_equal(got, want), mode
