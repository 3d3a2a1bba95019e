"""The reference's relaxed fast engine (eta > 0) on the
device against the reference library itself: kinetic_convolve(u, kernel, eta,
ConvEngine::Fast) and step_fully_discrete with its potential, values `==` and
block counts `==` (proj/src/minplus.cpp:152-276, proj/src/scheme.cpp:107-164).
For eta > 0 these are the reference's approximate values (relaxed merges of
48-capped blocks), reproduced bit for bit; eta == 0 is the exact engine."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api
from paper_1210_4090_b200._capi import InvalidInput

pytestmark = pytest.mark.gpu


def lines_of(kind, n, count, seed):
    rng = np.random.default_rng(seed)
    x = np.arange(n) / n
    out = []
    for l in range(count):
        if kind == "rough":  # C3-like Lipschitz random walk
            w = np.concatenate([[0.0], np.cumsum(rng.uniform(-1.0 / n, 1.0 / n, n))])
            out.append(w[:n] - w[n] * np.arange(n) / n)
        elif kind == "wiggle":  # cos + tiny wiggles (proj/tests/unit_minplus.cpp:307-315)
            out.append(np.cos(2 * np.pi * x) + 1e-9 * np.sin(2 * np.pi * 37 * x + l))
        elif kind == "fourier":  # C5-like modes
            k = rng.integers(1, 32, 16)
            ph = rng.uniform(0, 2 * np.pi, 16)
            out.append(sum(np.sin(2 * np.pi * kk * x + p) / kk ** 2 for kk, p in zip(k, ph)))
        else:  # random values
            out.append(rng.uniform(-1, 1, n))
    return np.stack(out)


def run(dev, u, tau, drifts, eta, tv=None):
    import torch

    lines, n = u.shape
    ks = [dev.build_kernel(n, tau, d) for d in drifts]
    kt = torch.from_numpy(np.concatenate([k.window for k in ks])).cuda()
    fr = torch.tensor([k.first for k in ks], dtype=torch.int64, device="cuda")
    du = torch.from_numpy(u).cuda()
    out = torch.empty_like(du)
    bl = torch.empty(lines, dtype=torch.int64, device="cuda")
    dtv = None if tv is None else torch.from_numpy(tv).cuda()
    dev.relaxed_f64(du, out, kt, fr, eta, tv=dtv, ktab_stride=2 * n + 1, blocks=bl)
    torch.cuda.synchronize()
    return out.cpu().numpy(), bl.cpu().numpy()


@pytest.mark.parametrize("eta", [0.0, 1e-9, 1e-6, 1e-4, 1e-2])
@pytest.mark.parametrize("kind,n,tau", [("rough", 128, 0.05), ("wiggle", 256, 0.05), ("fourier", 1024, 0.01),
                                        ("random", 24, 0.25), ("rough", 4096, 0.01)])
def test_relaxed_convolve_equals_reference(dev, ref, eta, kind, n, tau):
    drifts = [0.0, 0.4, -0.7, 1.0]
    u = lines_of(kind, n, len(drifts), n + int(eta * 1e9) % 97)
    got, blocks = run(dev, u, tau, drifts, eta)
    for l, d in enumerate(drifts):
        want, wb, st = ref.kinetic_convolve(u[l], n, tau, d, eta=eta, engine=0)
        assert st == 0
        assert np.array_equal(got[l], want), (kind, n, eta, d, np.max(np.abs(got[l] - want)))
        assert blocks[l] == wb


@pytest.mark.parametrize("eta", [0.0, 1e-5])
def test_relaxed_step_with_potential_equals_reference(dev, ref, eta):
    """step_fully_discrete(..., ConvEngine::Fast) with eta, C2-shaped drifts and V"""
    n, tau = 2048, 0.02
    drifts = api.gen_c2_drifts(256)[::37]
    v = api.gen_potential(2, n)
    u = lines_of("fourier", n, len(drifts), 11)
    got, blocks = run(dev, u, tau, drifts, eta, tv=np.ascontiguousarray(np.tile(api.tau_v(v, tau), (1, 1))[0]))
    want, wb = ref.step_lines(u, tau, drifts, v=v, eta=eta, engine=0, nthreads=4)
    assert np.array_equal(got, want)
    assert np.array_equal(blocks, wb)


def test_relaxed_equals_exact_at_eta_zero(dev, orc):
    """eta == 0: the fast engine is exact (proj/tests/unit_minplus.cpp:349-361) == K1"""
    n, tau = 512, 0.02
    u = lines_of("rough", n, 3, 5)
    drifts = [0.3, -1.2, 0.0]
    got, _ = run(dev, u, tau, drifts, 0.0)
    for l, d in enumerate(drifts):
        w, first, _, _ = orc.kernel(n, tau, d)
        assert np.array_equal(got[l], orc.direct(u[l:l + 1], w, first)[0])


def test_relaxed_evolution_tracks_reference(dev, ref):
    """ten relaxed steps in a row: every state == the reference's (errors would compound)"""
    n, tau, eta = 256, 0.05, 1e-4
    v = api.gen_potential(1, n)
    tv = np.ascontiguousarray(api.tau_v(v, tau))
    u = lines_of("fourier", n, 2, 3)
    drifts = [0.5, -0.25]
    for _ in range(10):
        got, _ = run(dev, u, tau, drifts, eta, tv=tv)
        want, _ = ref.step_lines(u, tau, drifts, v=v, eta=eta, engine=0)
        assert np.array_equal(got, want)
        u = got


def test_relaxed_argument_errors(dev):
    u = lines_of("random", 16, 1, 0)
    with pytest.raises(InvalidInput):
        run(dev, u, 0.25, [0.0], -1.0)
    bad = u.copy()
    bad[0, 3] = np.nan
    with pytest.raises(InvalidInput):
        run(dev, bad, 0.25, [0.0], 1e-3)


def test_relaxed_is_an_upper_bound_that_differs(dev, orc, ref):
    """eta > 0 exercises the approximation: values >= the exact minimum, some strictly
    (so the parity above is not the exact engine in disguise)"""
    n, tau = 1024, 0.01
    u = lines_of("rough", n, 2, 9)
    drifts = [0.0, 0.6]
    got, blocks = run(dev, u, tau, drifts, 1e-2)
    differs = 0
    for l, d in enumerate(drifts):
        w, first, _, _ = orc.kernel(n, tau, d)
        exact = orc.direct(u[l:l + 1], w, first)[0]
        assert np.all(got[l] >= exact)
        differs += int(np.sum(got[l] > exact))
        assert blocks[l] >= n // 48  # capped pieces
    assert differs > 0


@pytest.mark.parametrize("eta", [1e-6, 1e-3])
def test_relaxed_evolve_equals_reference(dev, ref, eta):
    """lob_evolve_f64 with LOB_ENGINE_RELAXED == the reference's evolve with ConvEngine::Fast and eta:
    final state and per-step block counts ==, per-step drift <= 1e-12 (device reduction order)"""
    import torch

    n, tau, steps, drift = 512, 0.02, 40, 0.7
    v = api.gen_potential(1, n)
    u0 = lines_of("fourier", n, 1, 21)[0]
    want_u, want_dr, want_bl, comp = ref.evolve(u0, tau, drift, v, steps, eta=eta, engine=0)
    assert comp
    du = torch.from_numpy(u0[None, :].copy()).cuda()
    scr = torch.empty_like(du)
    sd = torch.empty(steps, dtype=torch.float64, device="cuda")
    sb = torch.empty(steps, dtype=torch.int64, device="cuda")
    tv = torch.from_numpy(api.tau_v(v, tau)).cuda()
    dr = torch.tensor([drift], dtype=torch.float64, device="cuda")
    done = dev.evolve(du, scr, dr, tau, steps, tv=tv, eta=eta, engine=api.ENGINE_RELAXED, step_drift=sd,
                      step_blocks=sb)
    assert done == steps
    assert np.array_equal(du.cpu().numpy()[0], want_u)
    assert np.array_equal(sb.cpu().numpy(), want_bl)
    assert np.max(np.abs(sd.cpu().numpy() - want_dr)) <= 1e-12


def test_relaxed_host_step_equals_reference(dev, ref):
    n, tau, eta = 300, 0.05, 1e-4
    drifts = np.array([0.2, -0.9, 1.3])
    v = api.gen_potential(1, n)
    u = lines_of("rough", n, 3, 4)
    bl = np.empty(3, np.int64)
    got = dev.step_host(u, drifts, tau, tv=api.tau_v(v, tau), eta=eta, engine=api.ENGINE_RELAXED, blocks=bl)
    want, wb = ref.step_lines(u, tau, drifts, v=v, eta=eta, engine=0)
    assert np.array_equal(got, want)
    assert np.array_equal(bl, wb)


@pytest.mark.parametrize("eta", [0.0, 1e-6, 1e-2])
@pytest.mark.parametrize("n,tau", [(64, 0.1), (1000, 0.03)])
def test_relaxed_structured_inputs_equal_reference(dev, ref, eta, n, tau):
    """The adversarial shapes of tests/test_fast_gpu.py (constant, exact ties, jumps,
    1e8 magnitudes, spikes, near-ties) through the relaxed engine == the reference's
    ConvEngine::Fast: values and block counts."""
    from tests.test_fast_gpu import _structured_lines

    u = _structured_lines(n, np.random.default_rng(n + 1))
    drifts = list(np.linspace(-0.9, 1.3, u.shape[0]))
    got, blocks = run(dev, u, tau, drifts, eta)
    for l, d in enumerate(drifts):
        want, wb, st = ref.kinetic_convolve(u[l], n, tau, d, eta=eta, engine=0)
        assert st == 0
        assert np.array_equal(got[l], want), (l, eta, np.max(np.abs(got[l] - want)))
        assert blocks[l] == wb
