"""K1 (direct min-plus) parity on the B200 against the CPU oracle: bit-exact
(== per element; +0/-0 compare equal) at the BASELINE.json shapes."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=[api.DIRECT_SCREENED, api.DIRECT_PLAIN], ids=["screened", "plain"])
def direct_mode(request, dev):
    """Every K1 test runs with the fp32-screened sweep (default) and the plain fp64 sweep."""
    dev.set_direct_mode(request.param)
    yield request.param
    dev.set_direct_mode(api.DIRECT_SCREENED)


def torch_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def run_direct(dev, u, K, first, tv=None, ktab_stride=0, tv_stride=0):
    import torch
    lines = u.shape[0]
    du = torch_dev(u)
    out = torch.empty_like(du)
    dk = torch_dev(K)
    df = torch_dev(np.broadcast_to(np.asarray(first, np.int64), (lines,)).copy())
    dtv = None if tv is None else torch_dev(tv)
    dev.direct_f64(du, out, dk, df, tv=dtv, ktab_stride=ktab_stride, tv_stride=tv_stride)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("drift", [0.0, 0.4, -0.7, 1.0])
@pytest.mark.parametrize("n,tau", [(24, 0.25), (48, 0.125), (600, 0.04), (1024, 0.05)])
def test_direct_small_vs_oracle(dev, orc, n, tau, drift):
    # proj/tests/unit_scheme.cpp:176-194 at the reference's sizes and beyond
    rng = np.random.default_rng(39 + n)
    K, first, _, _ = orc.kernel(n, tau, drift)
    u = rng.uniform(-1, 1, (5, n))
    assert np.array_equal(run_direct(dev, u, K, first), orc.direct(u, K, first))


def test_direct_c3_lines_bit_exact(dev, orc):
    """C3: N=4096, tau=0.01, P=0, V=0; 32 of the 4096 seeded random-walk lines."""
    n = 4096
    K, first, _, _ = orc.kernel(n, 0.01, 0.0)
    u = api.gen_c3_lines(0, 32, n)
    got = run_direct(dev, u, K, first)
    want = orc.direct(u, K, first)
    assert np.array_equal(got, want)


def test_direct_c3_fp32_bit_exact(dev, orc):
    import torch
    n = 4096
    K, first, _, _ = orc.kernel(n, 0.01, 0.0)
    u = api.gen_c3_lines(100, 16, n).astype(np.float32)
    K32 = K.astype(np.float32)
    du, dk = torch_dev(u), torch_dev(K32)
    out = torch.empty_like(du)
    df = torch_dev(np.full(16, first, np.int64))
    dev.direct_f32(du, out, dk, df)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), orc.direct_f32(u, K32, first))


def test_direct_per_line_kernels_and_potential(dev, orc):
    """C2-like: per-line drift P_l (per-line tables, ktab_stride=W), shared tv."""
    n, tau = 2048, 0.02
    drifts = api.gen_c2_drifts(256)[::37]
    W = 2 * n + 1
    Ks, firsts = [], []
    for d in drifts:
        K, f, _, _ = orc.kernel(n, tau, d)
        Ks.append(K)
        firsts.append(f)
    Ks = np.concatenate(Ks)
    tv = api.tau_v(api.gen_potential(2, n), tau)
    rng = np.random.default_rng(5)
    u = np.cumsum(rng.uniform(-1.0 / n, 1.0 / n, (len(drifts), n)), axis=1)
    got = run_direct(dev, u, Ks, firsts, tv=tv, ktab_stride=W)
    want = np.stack([orc.direct(u[i:i + 1], Ks[i * W:(i + 1) * W], firsts[i], tv=tv)[0]
                     for i in range(len(drifts))])
    assert np.array_equal(got, want)


def test_windowed_lines(dev, orc):
    import torch
    n = 8
    K, first, _, _ = orc.kernel(n, 0.25, 0.0)
    rng = np.random.default_rng(40)
    u = rng.uniform(-1, 1, (3, 17))
    du = torch_dev(u)
    out = torch.empty_like(du)
    dev.window_f64(du, out, n, torch_dev(K), torch_dev(np.full(3, first, np.int64)))
    torch.cuda.synchronize()
    for l in range(3):
        want, st = orc.window(u[l], n, K, first)
        assert st == 0 and np.array_equal(out.cpu().numpy()[l], want)


def test_direct_properties_full_c3(dev, orc):
    """Size-independent properties on all 4096 C3 lines: constant-shift
    equivariance (proj/tests/unit_scheme.cpp:129-133, 1e-14) and
    non-expansiveness (:126-127)."""
    import torch
    n = 4096
    K, first, _, _ = orc.kernel(n, 0.01, 0.0)
    u = api.gen_c3_lines(0, 4096, n)
    a = run_direct(dev, u, K, first)
    b = run_direct(dev, u + 0.5, K, first)
    assert np.max(np.abs(b - (a + 0.5))) <= 1e-14
    v = u + np.random.default_rng(1).uniform(-1e-3, 1e-3, u.shape)
    c = run_direct(dev, v, K, first)
    assert np.max(np.abs(c - a)) <= np.max(np.abs(v - u)) + 1e-15
    # spot-check 8 random lines against the oracle bit-exactly
    idx = np.random.default_rng(2).choice(4096, 8, replace=False)
    assert np.array_equal(a[idx], orc.direct(u[idx], K, first))


def test_direct_screen_ties_fall_back_exactly(dev, orc, direct_mode):
    """Two equal wells half a period apart and a symmetric kernel: outputs a
    quarter period away see an exact tie between two sub-chunks, which the
    fp32 bound cannot separate; those outputs are swept in full fp64."""
    n = 4096
    K, first, _, _ = orc.kernel(n, 0.01, 0.0)
    u = np.zeros((2, n))
    u[:, 100] = u[:, 100 + n // 2] = -10.0  # deeper than K(+-n/4) = 3.125
    u[1] += np.linspace(0, 1e-9, n)  # breaks some ties below fp32 resolution
    dev.direct_fallbacks(reset=True)
    assert np.array_equal(run_direct(dev, u, K, first), orc.direct(u, K, first))
    if direct_mode == api.DIRECT_SCREENED:
        assert dev.direct_stats()["fp64_candidates"] > 0


@pytest.mark.parametrize("scale", [1e300, 1e-40, 1e-310])
def test_direct_screen_extreme_magnitudes(dev, orc, scale):
    """fp32 overflow (1e300: the CTA sweeps in fp64) and fp32/fp64 subnormal
    ranges (the bound's absolute slack) still give the reference's doubles."""
    n = 2048
    rng = np.random.default_rng(7)
    K, first, _, _ = orc.kernel(n, 0.02, 0.3)
    u = rng.uniform(-1, 1, (3, n)) * scale
    assert np.array_equal(run_direct(dev, u, K, first), orc.direct(u, K, first))
    Ks = K * scale
    assert np.array_equal(run_direct(dev, u, Ks, first), orc.direct(u, Ks, first))


def test_direct_screen_nan_inputs_match_reference_min(dev, orc):
    """NaN candidates never win std::min(best, c) (proj/src/minplus.cpp:121-123)."""
    n = 1024
    K, first, _, _ = orc.kernel(n, 0.05, 0.5)
    u = np.sin(np.linspace(0, 2 * np.pi, n, endpoint=False))[None, :].repeat(2, 0)
    u[0, 17] = np.nan
    got, want = run_direct(dev, u, K, first), orc.direct(u, K, first)
    assert np.array_equal(got, want, equal_nan=True)


@pytest.mark.parametrize("n", [2049, 4097, 515])
def test_direct_odd_lengths(dev, orc, n):
    """Odd n on the 16-output and 8-output register tilings (partial last tiles and chunks)."""
    rng = np.random.default_rng(n)
    K, first, _, _ = orc.kernel(n, 0.03, -0.4)
    u = np.cumsum(rng.uniform(-1.0 / n, 1.0 / n, (3, n)), axis=1)
    tv = rng.uniform(-1e-3, 1e-3, n)
    assert np.array_equal(run_direct(dev, u, K, first, tv=tv), orc.direct(u, K, first, tv=tv))
