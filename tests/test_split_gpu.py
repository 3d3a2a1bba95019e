"""K3 (2-D dimension splitting: transposes + sweeps + separable potential)
parity on the B200 against the oracle and the reference itself."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api

pytestmark = pytest.mark.gpu


FUSED = 100  # pseudo-engine of these tests: ENGINE_FAST with the two-half workspace (fused step)


def run_split(dev, u, tau, d1, d2, a1=None, a2=None, b=0.0, engine=api.ENGINE_DIRECT):
    import torch
    n = u.shape[0]
    du = torch.from_numpy(np.ascontiguousarray(u)).cuda()
    out = torch.empty_like(du)
    tmp = torch.empty_like(du)
    halves = 2 if engine == FUSED else 1
    engine = api.ENGINE_FAST if engine == FUSED else engine
    ws = torch.empty(halves * dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
    ta1 = None if a1 is None else torch.from_numpy(a1).cuda()
    ta2 = None if a2 is None else torch.from_numpy(a2).cuda()
    dev.split_step_2d(du, out, tmp, tau, d1, d2, a1=ta1, a2=ta2, b=b, engine=engine, workspace=ws)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("engine", [api.ENGINE_DIRECT, api.ENGINE_FAST, FUSED])
def test_split_16_vs_reference(dev, orc, ref, engine):
    # proj/tests/unit_splitting.cpp:103-121 / acceptance criterion 5
    rng = np.random.default_rng(42)
    n, tau = 16, 0.25
    for _ in range(5):
        u = rng.uniform(-1, 1, (n, n))
        got = run_split(dev, u, tau, 0.0, 0.5, engine=engine)
        assert np.array_equal(got, ref.split_step_2d(u, tau, 0.0, 0.5))


@pytest.mark.parametrize("engine", [api.ENGINE_DIRECT, api.ENGINE_FAST, FUSED])
def test_split_c4_potential_vs_reference(dev, ref, engine):
    """C4's kinetics and potential V = cos(2 pi x1) cos(2 pi x2) + 0.2 sin(2 pi t) at t+tau."""
    n, tau, t = 64, 0.05, 0.35
    u = api.gen_c4_u0(n)
    a = api.gen_cos(n)
    b = api.c4_time_term(t + tau)
    got = run_split(dev, u, tau, 0.3, -0.7, a1=a, a2=a, b=b, engine=engine)
    want = ref.split_step_2d(u, tau, 0.3, -0.7, pot_kind=1, t=t)
    assert np.array_equal(got, want)


def test_split_c4_full_size_vs_oracle(dev, orc):
    """C4 at full size (2048^2, tau=0.01, P=(0.3,-0.7)), one step, both engines
    bit-identical to the oracle's split step."""
    n, tau, t = 2048, 0.01, 0.0
    u = api.gen_c4_u0(n)
    a = api.gen_cos(n)
    b = api.c4_time_term(t + tau)
    k1, f1, _, _ = orc.kernel(n, tau, 0.3)
    k2, f2, _, _ = orc.kernel(n, tau, -0.7)
    tv = api.tau_v(np.add(np.multiply(a[:, None], a[None, :]), b), tau)
    want = orc.split2d(u, k1, f1, k2, f2, tv=tv)
    for engine in (api.ENGINE_DIRECT, api.ENGINE_FAST, FUSED):
        got = run_split(dev, u, tau, 0.3, -0.7, a1=a, a2=a, b=b, engine=engine)
        assert np.array_equal(got, want), engine


def test_split_separable_data_stays_separable(dev, orc):
    # proj/tests/unit_splitting.cpp:76-101: f(x1)+g(x2) -> (f conv K)(x1)+(g conv K)(x2), 1e-13
    rng = np.random.default_rng(41)
    n, tau = 16, 0.25
    f, g = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    u = f[:, None] + g[None, :]
    got = run_split(dev, u, tau, 0.0, 0.0)
    K, first, _, _ = orc.kernel(n, tau, 0.0)
    f1 = orc.direct(f[None, :], K, first)[0]
    g1 = orc.direct(g[None, :], K, first)[0]
    assert np.max(np.abs(got - (f1[:, None] + g1[None, :]))) <= 1e-13 * np.max(np.abs(got))


@pytest.mark.parametrize("engine", [api.ENGINE_DIRECT, api.ENGINE_FAST, FUSED])
@pytest.mark.parametrize("n", [100, 513])
def test_split_non_tile_multiple_sizes(dev, orc, ref, engine, n):
    """n not a multiple of the 32x32 transpose tile (and odd): == reference at 100, == oracle at 513."""
    tau, t = 0.02, 0.1
    u = api.gen_c4_u0(n)
    a = api.gen_cos(n)
    b = api.c4_time_term(t + tau)
    got = run_split(dev, u, tau, 0.3, -0.7, a1=a, a2=a, b=b, engine=engine)
    if n <= 128:
        want = ref.split_step_2d(u, tau, 0.3, -0.7, pot_kind=1, t=t)
    else:
        k1, f1, _, _ = orc.kernel(n, tau, 0.3)
        k2, f2, _, _ = orc.kernel(n, tau, -0.7)
        tv = api.tau_v(np.add.outer(a, np.zeros(n)) * a[None, :] + b, tau)
        want = orc.split2d(u, k1, f1, k2, f2, tv=tv)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("n", [33, 64, 250, 512])
def test_split_fast_layouts_vs_reference(dev, ref, mode, n):
    """Every 2-D layout of the fast engine's split step (lob_ctx_set_fast_line): 0 tiled kernels
    with carried statistics, 1 columns in place (strided), 2 transposes around K2L row sweeps (the
    default), 3 columns read / rows written, 4 columns exchanged through DSMEM in clusters of 8,
    5 columns read by 2-D TMA tensor maps (odd or non-multiple-of-8 sizes fall back to 2) ==
    the reference's split_step_nd with the C4 potential."""
    rng = np.random.default_rng(n + mode)
    tau, t = (0.05 if n <= 64 else 0.01), 0.35  # eps / tau < 1
    u = api.gen_c4_u0(n) + 0.01 * rng.uniform(-1, 1, (n, n))
    a = api.gen_cos(n)
    b = api.c4_time_term(t + tau)
    dev.set_fast_line(mode)
    try:
        got = run_split(dev, u, tau, 0.3, -0.7, a1=a, a2=a, b=b, engine=FUSED)
    finally:
        dev.set_fast_line(2)
    assert np.array_equal(got, ref.split_step_2d(u, tau, 0.3, -0.7, pot_kind=1, t=t))


@pytest.mark.parametrize("n", [2051, 2304, 4096])
def test_split_fast_beyond_the_whole_line_limit(dev, n):
    """n > 2048: the split step leaves the whole-line kernel for the tiled K2 (statistics-producing
    transposes, a last tile of 3 or 256 samples, an odd n without bulk copies).  Three steps of
    the fast engine, both workspace layouts, == the direct engine on every point."""
    import torch
    tau = 0.01
    u0 = torch.from_numpy(api.gen_c4_u0(n)).cuda()
    am = torch.from_numpy(api.gen_cos(n)).cuda()

    def run(engine, halves):
        u, o, t = u0.clone(), torch.empty_like(u0), torch.empty_like(u0)
        ws = torch.empty(halves * dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
        for i in range(3):
            dev.split_step_2d(u, o, t, tau, 0.3, -0.7, a1=am, a2=am, b=api.c4_time_term(i * tau + tau),
                              engine=engine, workspace=ws)
            u, o = o, u
        torch.cuda.synchronize()
        return u.cpu().numpy()

    want = run(api.ENGINE_DIRECT, 1)
    assert np.array_equal(run(api.ENGINE_FAST, 1), want)
    assert np.array_equal(run(api.ENGINE_FAST, 2), want)
