"""The reference's remaining known-answer and property tests for the stepping path
(SURVEY.md 8c), restated in this harness: first for the CPU checkers (oracle restatement and
the reference library, `-m "not gpu"`), then for the device engines (`-m gpu`).

  * a constant is a fixed point of the kinetic-only flow   (proj/tests/unit_scheme.cpp:87-94)
  * a representable drift lands exactly on -0.1             (proj/tests/unit_scheme.cpp:96-106)
  * monotone, non-expansive, shift-equivariant              (proj/tests/unit_scheme.cpp:108-135)
  * one wrapped period == three unrolled periods            (proj/tests/unit_scheme.cpp:137-154)
  * rotation invariance                                     (proj/tests/unit_scheme.cpp:156-174)
  * the split sweeps commute, V is applied once             (proj/tests/unit_splitting.cpp:143-194)
  * slope ties stay exact; every small tie-heavy convex x convex / convex x concave pair
    (> 30 000 cases) through conv_fast == conv_naive        (proj/tests/unit_minplus.cpp:241-248,410-464)
"""
import itertools

import numpy as np
import pytest

from paper_1210_4090_b200 import api


# ----------------------------------------------------------------------------- case generators
def tie_heavy_functions():
    """Every convex f (non-decreasing slopes) and concave g (non-increasing slopes) with one to
    four slopes from {-2,-1,0,1,2}, values starting at 0 (all sums exact), plus the one-point
    function: 126 convex and 126 concave sequences -> 126*126*2 = 31 752 pairs."""
    pool = [-2.0, -1.0, 0.0, 1.0, 2.0]
    convex, concave = [], []
    for depth in range(1, 5):
        for c in itertools.combinations_with_replacement(pool, depth):  # non-decreasing
            convex.append(np.concatenate([[0.0], np.cumsum(c)]))
            concave.append(np.concatenate([[0.0], np.cumsum(c[::-1])]))
    convex.append(np.zeros(1))
    concave.append(np.zeros(1))
    return convex, concave


def random_line(rng, n, amp=1.0):
    return rng.uniform(-amp, amp, n)


def approx(a, b, eps):
    """The reference tests' tolerance: |a - b| < eps (1 + max(|a|, |b|))."""
    a, b = np.asarray(a), np.asarray(b)
    return bool(np.all(np.abs(a - b) < eps * (1.0 + np.maximum(np.abs(a), np.abs(b)))))


# ----------------------------------------------------------------------------- CPU: the checkers
def _orc_step(orc, u, n, tau, drift, tv=None):
    w, first, _, _ = orc.kernel(n, tau, drift)
    return orc.direct(np.atleast_2d(u), w, np.array([first], np.int64), tv=tv)[0]


def test_checkers_constant_fixed_point_and_representable_drift(orc, ref):
    u = np.full(32, 1.25)
    assert np.array_equal(_orc_step(orc, u, 32, 0.125, 0.0), u)
    assert np.array_equal(ref.step_lines(u[None], 0.125, 0.0, engine=1)[0][0], u)
    # tau*P/eps = 2: the minimising displacement is on the grid, tau*K*(1) = -0.1 exactly
    z = np.zeros(10)
    assert np.array_equal(_orc_step(orc, z, 10, 0.2, 1.0), np.full(10, -0.1))
    for eng in (0, 1):
        assert np.array_equal(ref.step_lines(z[None], 0.2, 1.0, engine=eng)[0][0], np.full(10, -0.1))


def test_checkers_monotone_nonexpansive_shift_rotation(orc):
    rng = np.random.default_rng(31)
    n, tau, P = 64, 0.125, 0.5
    tv = tau * 0.7 * np.cos(2 * np.pi * np.arange(n) / n)
    for _ in range(20):
        u, v = random_line(rng, n), random_line(rng, n)
        su, sv = _orc_step(orc, u, n, tau, P, tv), _orc_step(orc, v, n, tau, P, tv)
        sup = _orc_step(orc, np.maximum(u, v), n, tau, P, tv)
        assert np.all(su <= sup + 1e-12)
        assert np.max(np.abs(su - sv)) <= np.max(np.abs(u - v)) + 1e-12
        assert approx(_orc_step(orc, u + 0.75, n, tau, P, tv), su + 0.75, 1e-14)
    # rotation by r samples (kinetic part only: the potential would rotate with the grid)
    u = random_line(rng, 48)
    s = _orc_step(orc, u, 48, 0.125, 0.3)
    assert np.array_equal(_orc_step(orc, np.roll(u, -17), 48, 0.125, 0.3), np.roll(s, -17))


def test_checkers_wrapped_period_equals_three_unrolled(orc, ref):
    rng = np.random.default_rng(32)
    n, tau, P = 32, 0.125, 0.4
    u = random_line(rng, n)
    stepped = _orc_step(orc, u, n, tau, P)
    tiled = np.concatenate([u, u, u, u[:1]])
    for who in ("oracle", "reference"):
        if who == "oracle":
            w, first, _, _ = orc.kernel(n, tau, P)
            got, st = orc.window(tiled, n, w, first)
            assert st == 0
        else:
            got, _, st = ref.kinetic_convolve(tiled, n, tau, P, engine=1, periodic=False)
            assert st == 0
        assert np.array_equal(got[n:2 * n + 1], np.concatenate([stepped, stepped[:1]])), who


def test_checkers_split_commutes_and_applies_v_once(orc):
    rng = np.random.default_rng(44)
    n, tau = 16, 0.25
    u = rng.uniform(-1, 1, (n, n))
    k1, f1, _, _ = orc.kernel(n, tau, 0.25)
    k2, f2, _, _ = orc.kernel(n, tau, -0.5)
    out = orc.split2d(u, k1, f1, k2, f2)
    outt = orc.split2d(np.ascontiguousarray(u.T), k2, f2, k1, f1)
    assert approx(out, outt.T, 1e-14)
    k0, f0, _, _ = orc.kernel(n, tau, 0.0)
    x = np.arange(n) / n
    v = x[:, None] + 2.0 * x[None, :]
    a = orc.split2d(u, k0, f0, k0, f0)
    b = orc.split2d(u, k0, f0, k0, f0, tv=tau * v)
    assert np.array_equal(b, a - tau * v)  # one subtraction of the rounded product


def test_reference_fast_equals_naive_on_every_tie_heavy_pair(orc, ref):
    """The exhaustive engine equality the reference asserts for itself, re-run here against its
    library and with the oracle's conv_naive as the third witness."""
    convex, concave = tie_heavy_functions()
    assert np.array_equal(ref.conv(2, [0.0, 0.0, 1.0, 3.0], [0.0, 1.0, 1.0])[0],
                          ref.conv(0, [0.0, 0.0, 1.0, 3.0], [0.0, 1.0, 1.0])[0])
    cases = 0
    for f in convex:
        for which, others in ((1, convex), (2, concave)):
            for g in others:
                want = orc.conv_naive(f, g)
                assert np.array_equal(ref.conv(0, f, g)[0], want)
                assert np.array_equal(ref.conv(which, f, g)[0], want)
                assert np.array_equal(ref.conv(3, f, g)[0], want)
                cases += 1
    assert cases > 30000


# ----------------------------------------------------------------------------- GPU: the engines
def _to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float64)).cuda()


def _dev_steps(dev, u, tau, drift, tv=None):
    """One step of the lines u (lines x n, one drift) through K1 screened / plain, K2 (whole-line and
    tiled), the window-table K2 and the relaxed engine at eta = 0."""
    import torch
    u = np.atleast_2d(u)
    lines, n = u.shape
    du = _to_dev(u)
    k = dev.build_kernel(n, tau, drift)
    kt = _to_dev(k.window)
    fr = torch.full((lines,), int(k.first), dtype=torch.int64, device="cuda")  # one per line
    dtv = None if tv is None else _to_dev(tv)
    dd = _to_dev(np.full(lines, drift))
    res = {}
    for name, mode in (("k1_screened", api.DIRECT_SCREENED), ("k1_plain", api.DIRECT_PLAIN)):
        dev.set_direct_mode(mode)
        o = torch.empty_like(du)
        dev.direct_f64(du, o, kt, fr, tv=dtv)
        res[name] = o
    dev.set_direct_mode(api.DIRECT_SCREENED)
    for name, mode in (("k2_line", 2), ("k2_tiled", 0)):
        dev.set_fast_line(mode)
        ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
        o = torch.empty_like(du)
        dev.fast_f64(du, o, dd, tau, tv=dtv, workspace=ws)
        res[name] = o
    dev.set_fast_line(2)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    o = torch.empty_like(du)
    dev.fast_window_f64(du, o, kt, fr, tau, tv=dtv, workspace=ws)
    res["k2_window"] = o
    o = torch.empty_like(du)
    dev.relaxed_f64(du, o, kt, fr, 0.0, tv=dtv)
    res["relaxed"] = o
    torch.cuda.synchronize()
    return {name: v.cpu().numpy() for name, v in res.items()}


@pytest.mark.gpu
def test_device_constant_fixed_point_and_representable_drift(dev):
    u = np.full((3, 32), 1.25)
    for name, got in _dev_steps(dev, u, 0.125, 0.0).items():
        assert np.array_equal(got, u), name
    for name, got in _dev_steps(dev, np.zeros((2, 10)), 0.2, 1.0).items():
        assert np.array_equal(got, np.full((2, 10), -0.1)), name


@pytest.mark.gpu
def test_device_monotone_nonexpansive_shift_rotation(dev):
    rng = np.random.default_rng(31)
    n, tau, P = 64, 0.125, 0.5
    tv = tau * 0.7 * np.cos(2 * np.pi * np.arange(n) / n)
    u, v = rng.uniform(-1, 1, (20, n)), rng.uniform(-1, 1, (20, n))
    su, sv = _dev_steps(dev, u, tau, P, tv), _dev_steps(dev, v, tau, P, tv)
    sup = _dev_steps(dev, np.maximum(u, v), tau, P, tv)
    lifted = _dev_steps(dev, u + 0.75, tau, P, tv)
    for name in su:
        assert np.all(su[name] <= sup[name] + 1e-12), name
        assert np.all(np.max(np.abs(su[name] - sv[name]), axis=1) <= np.max(np.abs(u - v), axis=1) + 1e-12), name
        assert approx(lifted[name], su[name] + 0.75, 1e-14), name
    w = rng.uniform(-1, 1, (4, 48))
    s, sr = _dev_steps(dev, w, 0.125, 0.3), _dev_steps(dev, np.roll(w, -17, axis=1), 0.125, 0.3)
    for name in s:
        assert np.array_equal(sr[name], np.roll(s[name], -17, axis=1)), name


@pytest.mark.gpu
def test_device_wrapped_period_equals_three_unrolled(dev):
    import torch
    rng = np.random.default_rng(32)
    n, tau, P = 32, 0.125, 0.4
    u = rng.uniform(-1, 1, (5, n))
    stepped = _dev_steps(dev, u, tau, P)
    tiled = np.concatenate([u, u, u, u[:, :1]], axis=1)
    k = dev.build_kernel(n, tau, P)
    o = torch.empty((5, 3 * n + 1), dtype=torch.float64, device="cuda")
    dev.window_f64(_to_dev(tiled), o, n, _to_dev(k.window), torch.full((5,), int(k.first), dtype=torch.int64, device="cuda"))
    torch.cuda.synchronize()
    mid = o.cpu().numpy()[:, n:2 * n + 1]
    for name, s in stepped.items():
        assert np.array_equal(mid, np.concatenate([s, s[:, :1]], axis=1)), name


@pytest.mark.gpu
@pytest.mark.parametrize("engine", [api.ENGINE_DIRECT, api.ENGINE_FAST])
def test_device_split_commutes_and_applies_v_once(dev, engine):
    import torch
    rng = np.random.default_rng(44)
    n, tau = 16, 0.25
    u = rng.uniform(-1, 1, (n, n))

    def split(x, d1, d2, tv=None):
        dx = _to_dev(x)
        out, tmp = torch.empty_like(dx), torch.empty_like(dx)
        ws = torch.empty(2 * dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
        dev.split_step_nd(dx.view(-1), out.view(-1), tmp.view(-1), 2, n, tau,
                          kernels=[dev.build_kernel(n, tau, d1), dev.build_kernel(n, tau, d2)], drifts=[d1, d2],
                          tv=None if tv is None else _to_dev(tv).view(-1), engine=engine, workspace=ws)
        torch.cuda.synchronize()
        return out.cpu().numpy()

    out = split(u, 0.25, -0.5)
    outt = split(np.ascontiguousarray(u.T), -0.5, 0.25)
    assert approx(out, outt.T, 1e-14)
    x = np.arange(n) / n
    v = x[:, None] + 2.0 * x[None, :]
    a, b = split(u, 0.0, 0.0), split(u, 0.0, 0.0, tv=tau * v)
    assert np.array_equal(b, a - tau * v)


@pytest.mark.gpu
def test_device_conv_fast_equals_naive_on_tie_heavy_pairs(dev, orc, ref):
    """Every 7th of the 31 752 tie-heavy pairs (one-sample functions included) and the slope-tie
    known answer through the device's conv_fast and conv_naive == the oracle's conv_naive; the
    block count == the reference's conv_fast."""
    import torch
    convex, concave = tie_heavy_functions()

    def fast(a, b):
        out = torch.empty(len(a) + len(b) - 1, dtype=torch.float64, device="cuda")
        blocks = dev.conv_fast(_to_dev(a), _to_dev(b), out, 0.0)
        return out.cpu().numpy(), blocks

    def naive(a, b):
        out = torch.empty(len(a) + len(b) - 1, dtype=torch.float64, device="cuda")
        dev.conv_naive(_to_dev(a), _to_dev(b), out)
        return out.cpu().numpy()

    f, g = [0.0, 0.0, 1.0, 3.0], [0.0, 1.0, 1.0]
    assert np.array_equal(fast(f, g)[0], orc.conv_naive(f, g))
    pairs = [(f, g) for f in convex for g in convex + concave]
    assert len(pairs) > 30000
    one = np.zeros(1)
    for f, g in pairs[::7] + [(one, one), (one, convex[5]), (one, concave[9]), (convex[40], one)]:
        want = orc.conv_naive(f, g)
        got, blocks = fast(f, g)
        assert np.array_equal(got, want)
        _, want_blocks, st = ref.conv(3, f, g)
        assert st == 0 and blocks == want_blocks
        assert np.array_equal(naive(f, g), want)


@pytest.mark.gpu
def test_device_conv_fast_rejects_a_non_convex_kernel_like_the_reference(dev, ref):
    """conv_fast(kernel, u, eta) requires a convex kernel (require_convex,
    proj/src/minplus.cpp:24-29,190-194): InvalidInput naming the first segment whose slope drops."""
    import torch
    bad = np.array([0.0, 1.0, 3.0, 4.0, 4.5, 7.0])  # slopes 1, 2, 1, 0.5, 2.5: first drop after segment 2
    u = np.array([0.0, 1.0, 0.5])
    assert ref.conv(3, bad, u)[2] != 0
    assert "segment 2" in ref.err()
    out = torch.empty(len(bad) + len(u) - 1, dtype=torch.float64, device="cuda")
    with pytest.raises(api.InvalidInput, match="not convex, slope drops at segment 2"):
        dev.conv_fast(_to_dev(bad), _to_dev(u), out, 0.0)
    ok = np.array([0.0, 1.0, 3.0, 6.0])
    out = torch.empty(len(ok) + len(u) - 1, dtype=torch.float64, device="cuda")
    dev.conv_fast(_to_dev(ok), _to_dev(u), out, 0.0)
    assert np.array_equal(out.cpu().numpy(), ref.conv(0, ok, u)[0])
