"""Weak-KAM consumers of the step (proj/src/weakkam.cpp):
min-plus products, the one-period matrix, Karp's eigenvalue and the drift
estimator, checked against the reference library itself (oracle/_ref) on the
same inputs.  The reference's own tests (proj/tests/unit_weakkam.cpp,
proj/tests/acceptance.cpp:316-366) are re-expressed here; potentials are
tables (the same doubles on both sides), so every comparison is `==`.

CPU tests pin the host helpers and the reference's known answers; GPU tests
run the device kernels through the C-ABI."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api
from paper_1210_4090_b200._capi import InvalidInput

INF = np.inf


def cos_table(n, offset=1.0, amp=-1.0, freq=1, phase=0.0):
    """offset + amp*cos(freq*2*pi*x_j + phase) sampled on the grid (a table potential)."""
    x = np.arange(n) / n
    return offset + amp * np.cos(freq * 2.0 * np.pi * x + phase)


def cosine_u0(n, freq):
    # proj/tests/unit_weakkam.cpp:32-37 (theta(x) = 2 pi x - pi)
    x = np.arange(n) * (1.0 / n)
    return np.cos(freq * (2.0 * np.pi * x - np.pi))


def tv_tables(vtabs, tau):
    """The device's per-step tables: step i of a period samples V at t_i + tau
    (Arrival), i.e. table (i + 1) mod ell of the reference's time-indexed tables."""
    v = np.atleast_2d(vtabs)
    if v.shape[0] == 1:
        return tau * v
    return tau * np.roll(v, -1, axis=0)


def brute_min_cycle_mean(c):
    """Exhaustive minimum simple-cycle mean (proj/tests/unit_weakkam.cpp:39-60)."""
    n = c.shape[0]
    best = INF

    def dfs(start, at, cost, arcs, used):
        nonlocal best
        best = min(best, (cost + c[at, start]) / (arcs + 1))
        for nxt in range(n):
            if nxt in used or nxt == start:
                continue
            used.add(nxt)
            dfs(start, nxt, cost + c[at, nxt], arcs + 1, used)
            used.discard(nxt)

    for s in range(n):
        dfs(s, s, 0.0, 0, set())
    return best


# ---------------------------------------------------------------- CPU ------

@pytest.mark.parametrize("n,drift", [(16, 0.0), (17, 0.4), (32, -1.3), (9, 2.0)])
def test_period_kinetic_host_equals_reference_row(ref, n, drift):
    """lob_period_kinetic_host == row 0 of the reference's one-step period matrix (tau = 1, V = 0)."""
    w, first, arg, st = ref.kernel(n, 1.0, drift)
    assert st == 0
    kinc = api.Device.period_kinetic(api.Kernel(w, first, arg, first + n, n, 1.0, drift))
    c = ref.period_matrix(n, 1.0, drift)
    assert np.array_equal(kinc, c[0])
    # translation invariance (proj/tests/unit_weakkam.cpp:102-112)
    for y in range(n):
        assert np.array_equal(c[y], np.roll(kinc, y))


def test_reference_karp_known_answers(ref):
    """The oracle is pinned to the reference's KATs (proj/tests/unit_weakkam.cpp:149-169)."""
    assert ref.karp(np.zeros((5, 5)))[0] == 0.0
    assert ref.karp(np.array([[0.0, 5.0], [1.0, 0.0]]))[0] == 0.0
    rng = np.random.default_rng(53)
    for _ in range(5):
        m = rng.uniform(-2, 2, (6, 6))
        assert ref.karp(m)[0] == pytest.approx(brute_min_cycle_mean(m), rel=1e-12, abs=1e-14)
    assert ref.karp(np.array([[0.0, INF], [1.0, 0.0]]))[1] == 1  # InvalidInput


def test_reference_drift_known_answers(ref):
    """proj/tests/unit_weakkam.cpp:66-100 through the reference itself."""
    r = ref.hbar_drift(cosine_u0(32, 2), 0.1, 0.0, None, 200, 1e-10)
    assert r["converged"] and abs(r["h_bar"]) <= 1e-13
    c = 0.8125
    r = ref.hbar_drift(cosine_u0(32, 1), 0.1, 0.0, np.full(32, c), 200, 1e-10)
    assert r["converged"] and r["h_bar"] == pytest.approx(-c, rel=1e-12)
    r = ref.hbar_drift(np.zeros(10), 0.2, 1.0, None, 100, 1e-10)
    assert r["converged"] and r["h_bar"] == pytest.approx(-0.5, rel=1e-12)
    assert ref.hbar_drift(cosine_u0(32, 1), 0.15, 0.0, None, 10, 1e-8)["status"] == 1


# ---------------------------------------------------------------- GPU ------

def _cuda(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def _host(t):
    import torch

    torch.cuda.synchronize()
    return t.cpu().numpy()


def _gemm(dev, a, b):
    import torch

    da, db = _cuda(a), _cuda(b)
    out = torch.empty((a.shape[0], b.shape[1]), dtype=torch.float64, device="cuda")
    dev.minplus_gemm(da, db, out)
    return _host(out)


def tie_heavy(rng, shape):
    """small integers and halves with signed zeros and infinities: exact ties everywhere"""
    m = rng.integers(-3, 4, shape).astype(np.float64) * 0.5
    m[rng.random(shape) < 0.1] = -0.0
    m[rng.random(shape) < 0.03] = INF
    return m


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 12, 31, 64, 200, 512, 700])
def test_minplus_product_equals_reference(dev, ref, n):
    rng = np.random.default_rng(52 + n)
    for a, b in [(rng.uniform(-1, 1, (n, n)), rng.uniform(-1, 1, (n, n))),
                 (tie_heavy(rng, (n, n)), tie_heavy(rng, (n, n)))]:
        want = ref.minplus_product(a, b)
        got = _gemm(dev, a, b)
        assert np.array_equal(got, want, equal_nan=True)
        # the sign of zero survives exactly like the reference's first-minimum rule
        assert np.array_equal(np.signbit(got), np.signbit(want))


@pytest.mark.gpu
def test_minplus_product_negative_infinity(dev, ref):
    """inf + -inf candidates are NaN and ignored on both sides"""
    rng = np.random.default_rng(7)
    a = rng.uniform(-1, 1, (40, 40))
    b = rng.uniform(-1, 1, (40, 40))
    a[3, :] = INF
    b[:, 5] = -INF
    b[7, 9] = -INF
    want = ref.minplus_product(a, b)
    got = _gemm(dev, a, b)
    assert np.array_equal(got, want, equal_nan=True)


@pytest.mark.gpu
@pytest.mark.parametrize("n,lines", [(48, 1), (100, 7), (256, 33)])
def test_minplus_apply_equals_reference(dev, ref, n, lines):
    rng = np.random.default_rng(n)
    cm = rng.uniform(-1, 1, (n, n))
    u = rng.uniform(-1, 1, (lines, n))
    got = _gemm(dev, u, cm)
    for l in range(lines):
        assert np.array_equal(got[l], ref.minplus_apply(cm, u[l]))


def _device_period_matrix(dev, n, tau, drift, vtabs):
    import torch

    ell = int(round(1.0 / tau))
    k = dev.build_kernel(n, tau, drift)
    kinc = _cuda(api.Device.period_kinetic(k))
    tvs = None
    if vtabs is not None:
        v = np.atleast_2d(vtabs)
        tv = tv_tables(v, tau)
        tvs = _cuda(np.repeat(tv, ell, axis=0) if v.shape[0] == 1 else tv)
    out = torch.empty((n, n), dtype=torch.float64, device="cuda")
    scratch = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
    dev.period_matrix(kinc, tvs, ell, out, scratch)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("n,tau,drift,kind", [
    (16, 1.0, 0.0, "zero"),     # proj/tests/unit_weakkam.cpp:102-112
    (32, 0.2, 1.0, "cos"),      # :114-130
    (32, 0.125, 0.0, "cos"),    # :172-192 cases
    (48, 0.125, 1.0, "cos"),
    (64, 0.1, 0.5, "cos2"),
    (40, 0.25, -0.6, "timedep"),
    (128, 0.125, 0.3, "timedep"),
])
def test_period_matrix_equals_reference(dev, ref, n, tau, drift, kind):
    ell = int(round(1.0 / tau))
    vt = {"zero": None, "cos": cos_table(n), "cos2": cos_table(n, 0.5, 0.5, 2),
          "timedep": np.stack([cos_table(n, 0.2 * i, -1.0 + 0.1 * i, 1 + i % 3) for i in range(ell)])}[kind]
    want = ref.period_matrix(n, tau, drift, vt)
    got = _host(_device_period_matrix(dev, n, tau, drift, vt))
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_karp_known_answers_and_errors(dev, ref):
    assert dev.eigenvalue_karp(_cuda(np.zeros((5, 5)))) == 0.0
    assert dev.eigenvalue_karp(_cuda(np.array([[0.0, 5.0], [1.0, 0.0]]))) == 0.0
    with pytest.raises(InvalidInput):
        dev.eigenvalue_karp(_cuda(np.array([[0.0, INF], [1.0, 0.0]])))
    with pytest.raises(InvalidInput):
        dev.eigenvalue_karp(_cuda(np.array([[np.nan]])))


@pytest.mark.gpu
@pytest.mark.parametrize("n,reps", [(1, 3), (8, 25), (33, 4), (128, 2), (512, 1), (600, 1)])
def test_karp_equals_reference(dev, ref, n, reps):
    rng = np.random.default_rng(53 + n)
    for _ in range(reps):
        m = rng.uniform(-2, 2, (n, n))
        want, st = ref.karp(m)
        assert st == 0
        assert dev.eigenvalue_karp(_cuda(m)) == want
        if n <= 8:
            assert want == pytest.approx(brute_min_cycle_mean(m), rel=1e-12, abs=1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("n,tau,drift,kind", [(32, 0.125, 0.0, "cos"), (48, 0.125, 1.0, "cos"),
                                              (64, 0.1, 0.5, "cos2"), (40, 0.25, -0.6, "timedep")])
def test_karp_of_period_matrix_equals_reference(dev, ref, n, tau, drift, kind):
    """eigenvalue_karp(build_period_matrix(...)) end to end (proj/tests/unit_weakkam.cpp:172-192)."""
    ell = int(round(1.0 / tau))
    vt = {"cos": cos_table(n), "cos2": cos_table(n, 0.5, 0.5, 2),
          "timedep": np.stack([cos_table(n, 0.2 * i, -1.0 + 0.1 * i, 1 + i % 3) for i in range(ell)])}[kind]
    want, st = ref.karp(ref.period_matrix(n, tau, drift, vt))
    assert st == 0
    assert dev.eigenvalue_karp(_device_period_matrix(dev, n, tau, drift, vt)) == want


@pytest.mark.gpu
@pytest.mark.parametrize("engine", [api.ENGINE_FAST, api.ENGINE_DIRECT])
@pytest.mark.parametrize("case", [
    ("flat", 32, 0.1, 0.0, None, 2, 200, 1e-10),          # proj/tests/unit_weakkam.cpp:66-74
    ("const", 32, 0.1, 0.0, "const", 1, 200, 1e-10),      # :76-84
    ("drift", 10, 0.2, 1.0, None, 0, 100, 1e-10),         # :86-93
    ("cos", 32, 0.125, 0.0, "cos", 2, 600, 1e-8),         # :172-192
    ("cos-drift", 48, 0.125, 1.0, "cos", 2, 600, 1e-8),
    ("cos2", 64, 0.1, 0.5, "cos2", 2, 600, 1e-8),
    ("timedep", 40, 0.25, -0.6, "timedep", 1, 300, 1e-9),
])
def test_hbar_drift_equals_reference(dev, ref, engine, case):
    name, n, tau, drift, kind, freq, periods, tol = case
    ell = int(round(1.0 / tau))
    u0 = np.zeros(n) if freq == 0 else cosine_u0(n, freq)
    vt = {None: None, "const": np.full(n, 0.8125), "cos": cos_table(n), "cos2": cos_table(n, 0.5, 0.5, 2),
          "timedep": np.stack([cos_table(n, 0.2 * i, -1.0 + 0.1 * i, 1 + i % 3) for i in range(ell)])}[kind]
    want = ref.hbar_drift(u0, tau, drift, vt, periods, tol)
    assert want["status"] == 0
    got = dev.hbar_drift_host(u0, drift, tau, None if vt is None else tv_tables(vt, tau), engine, periods, tol)
    for key in ("h_bar", "residual", "n_steps", "converged"):
        assert got[key] == want[key], (name, key, got[key], want[key])
    # fixed_point_residual at the estimate (proj/src/weakkam.cpp:191-201)
    r_want, st = ref.fixed_point_residual(got["u"], tau, drift, want["h_bar"], vt)
    assert st == 0
    r_got = dev.fixed_point_residual_host(got["u"], drift, tau, want["h_bar"],
                                          None if vt is None else tv_tables(vt, tau), engine)
    assert r_got == r_want


@pytest.mark.gpu
def test_hbar_drift_argument_errors(dev):
    u0 = cosine_u0(32, 1)
    with pytest.raises(InvalidInput):  # tau does not divide the period (unit_weakkam.cpp:95-100)
        dev.hbar_drift_host(u0, 0.0, 0.15, None, api.ENGINE_FAST, 10, 1e-8)
    with pytest.raises(InvalidInput):
        dev.hbar_drift_host(u0, 0.0, 0.125, None, api.ENGINE_FAST, 0, 1e-8)
    with pytest.raises(InvalidInput):  # 3 tables for 8 steps per period
        dev.hbar_drift_host(u0, 0.0, 0.125, np.zeros((3, 32)), api.ENGINE_FAST, 10, 1e-8)
