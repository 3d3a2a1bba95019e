"""step_semidiscrete (proj/src/scheme.cpp:166-206) against
the reference library itself (oracle/_ref).  The reference's own tests
(proj/tests/unit_scheme.cpp:196-250) are re-expressed.

Tolerances: Zero and Const potentials involve no transcendental function, so
the device result is `==` the reference's.  The Cosine potential's spatial
cos is the device's (CUDA double cos, <= 2 ulp) instead of glibc's, so those
cases are compared at |gpu - ref| <= 1e-12 * max(1, max|u|) (the north-star
fp64 tolerance)."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api
from paper_1210_4090_b200._capi import EvaluationError, InvalidInput

TOL = 1e-12


def random_line(rng, n, amp=1.0):
    return rng.uniform(-amp, amp, n)


# ---------------------------------------------------------------- CPU ------

def test_reference_semidiscrete_zero_potential_is_the_full_step(ref):
    """unit_scheme.cpp:209-220: with V = 0 the semi-discrete step is the kinetic convolution."""
    rng = np.random.default_rng(34)
    u = random_line(rng, 24)
    want, _, st = ref.kinetic_convolve(u, 24, 0.25, 0.25)
    assert st == 0
    got, st = ref.step_semidiscrete(u, 24, 0.25, 0.25, api.potential_zero(), 0.0, 4)
    assert st == 0
    assert np.array_equal(got, want)
    assert ref.step_semidiscrete(u, 24, 0.25, 0.25, api.potential_zero(), 0.0, 0)[1] == 1  # InvalidInput


# ---------------------------------------------------------------- GPU ------

def _run(dev, u, n, tau, drift, pot, t, q, periodic=True, origin=0.0):
    import torch

    k = dev.build_kernel(n, tau, drift)
    du = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(u))).cuda()
    out = torch.empty_like(du)
    kt = torch.from_numpy(k.window).cuda()
    dev.step_semidiscrete(du, out, kt, k.first, t, tau, pot, q, periodic, origin, n_space=n)
    torch.cuda.synchronize()
    return out.cpu().numpy()


POTS = {
    "zero": api.potential_zero(),
    "const": api.potential_const(0.8125),
    "const-neg": api.potential_const(-1.3),
    "cos": api.potential_cosine(0.0, 0.5, 1),
    "cos3": api.potential_cosine(0.2, -0.7, 3),
    "cos-sin": api.potential_cosine(0.0, 1.0, 2, api._capi.TMOD_SIN, 6.0),
    "cos-cos": api.potential_cosine(0.5, 0.5, 1, api._capi.TMOD_COS, 2.0 * np.pi),
}


@pytest.mark.gpu
@pytest.mark.parametrize("pot", list(POTS))
@pytest.mark.parametrize("n,tau,drift,q,t", [(24, 0.25, 0.25, 4, 0.0), (32, 0.25, 0.0, 1, 0.0),
                                             (16, 0.25, 0.0, 8, 0.2), (64, 0.05, -0.7, 3, 1.3),
                                             (128, 0.02, 1.1, 2, 0.0)])
def test_semidiscrete_periodic_equals_reference(dev, ref, pot, n, tau, drift, q, t):
    rng = np.random.default_rng(n + q)
    lines = 3
    u = np.stack([random_line(rng, n, 0.5) for _ in range(lines)])
    got = _run(dev, u, n, tau, drift, POTS[pot], t, q)
    for l in range(lines):
        want, st = ref.step_semidiscrete(u[l], n, tau, drift, POTS[pot], t, q)
        assert st == 0
        if POTS[pot]["kind"] == api._capi.POTENTIAL_COSINE:
            assert np.max(np.abs(got[l] - want)) <= TOL * max(1.0, np.max(np.abs(u[l])))
        else:
            assert np.array_equal(got[l], want)


@pytest.mark.gpu
@pytest.mark.parametrize("pot", ["zero", "const", "cos3"])
def test_semidiscrete_windowed_equals_reference(dev, ref, pot):
    """windowed domain (unit_scheme.cpp:196-207: n = 8, tau = 0.25, 17 samples from -1)"""
    rng = np.random.default_rng(40)
    for n, m, drift, origin in [(8, 17, 0.0, -1.0), (16, 40, 0.5, 0.25), (12, 7, -0.3, 0.0)]:
        u = rng.uniform(-1, 1, m)
        got = _run(dev, u, n, 0.25, drift, POTS[pot], 0.0, 2, periodic=False, origin=origin)[0]
        want, st = ref.step_semidiscrete(u, n, 0.25, drift, POTS[pot], 0.0, 2, periodic=False, origin=origin)
        assert st == 0
        if pot.startswith("cos"):
            assert np.max(np.abs(got - want)) <= TOL * max(1.0, np.max(np.abs(u)))
        else:
            assert np.array_equal(got, want)


@pytest.mark.gpu
def test_semidiscrete_zero_potential_is_the_direct_step(dev, orc):
    """unit_scheme.cpp:209-220 on the device: semi-discrete(V = 0) == K1 step, bit for bit"""
    rng = np.random.default_rng(34)
    for n, tau, drift in [(24, 0.25, 0.25), (300, 0.01, 0.9)]:
        u = rng.uniform(-1, 1, (2, n))
        got = _run(dev, u, n, tau, drift, POTS["zero"], 0.0, 4)
        w, first, _, _ = orc.kernel(n, tau, drift)
        assert np.array_equal(got, orc.direct(u, w, first))


@pytest.mark.gpu
def test_semidiscrete_trapezoid_second_order(dev):
    """unit_scheme.cpp:235-250: errors against q = 1024 halve (at least) with q"""
    rng = np.random.default_rng(36)
    u = rng.uniform(-0.5, 0.5, 16)
    pot = api.potential_cosine(0.0, 1.0, 2, api._capi.TMOD_SIN, 6.0)
    with pytest.raises(InvalidInput):  # the device handles q <= 64
        _run(dev, u, 16, 0.25, 0.0, pot, 0.2, 1024)
    refq = _run(dev, u, 16, 0.25, 0.0, pot, 0.2, 64)[0]
    prev = np.inf
    for q in (1, 2, 4, 8):
        err = np.max(np.abs(_run(dev, u, 16, 0.25, 0.0, pot, 0.2, q)[0] - refq))
        if prev < np.inf:
            assert err <= 0.5 * prev + 1e-13
        prev = err


@pytest.mark.gpu
def test_semidiscrete_endpoint_error_bound(dev, orc):
    """unit_scheme.cpp:222-233: |semi - full| <= tau * Lip(V)"""
    rng = np.random.default_rng(35)
    n, tau = 32, 0.25
    u = rng.uniform(-0.5, 0.5, n)
    pot = api.potential_cosine(0.0, 0.5, 1)
    semi = _run(dev, u, n, tau, 0.0, pot, 0.0, 8)[0]
    # the full step with V sampled at arrival: V(t + tau, x_j) = 0.5 cos(theta(x_j))
    x = np.arange(n) / n
    v = 0.5 * np.cos(2.0 * np.pi * x - np.pi)
    w, first, _, _ = orc.kernel(n, tau, 0.0)
    full = orc.direct(u[None, :], w, first, tv=tau * v)[0]
    assert np.max(np.abs(full - semi)) <= tau * 0.5 * 2.0 * np.pi + 1e-9


@pytest.mark.gpu
def test_semidiscrete_errors(dev, ref):
    u = np.zeros(8)
    with pytest.raises(InvalidInput):
        _run(dev, u, 8, 0.25, 0.0, None, 0.0, 0)
    # a windowed output with no source inside the domain (tau P / eps = 8 > the domain)
    u = np.zeros(4)
    with pytest.raises(EvaluationError):
        _run(dev, u, 4, 0.5, 4.0, None, 0.0, 1, periodic=False)
    assert ref.step_semidiscrete(u, 4, 0.5, 4.0, api.potential_zero(), 0.0, 1, periodic=False)[1] == 2
