"""Pin the C restatement oracle (oracle/laxol_oracle.c) to the reference
itself (oracle/_ref, built from /root/reference sources) and to the
reference's own known-answer tests.  CPU only."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api

RNG = np.random.default_rng


def rand_periodic(rng, n, amp=1.0):
    return rng.uniform(-amp, amp, n)


# ---- kernel build -----------------------------------------------------------

@pytest.mark.parametrize("n,tau,drift", [(100, 0.1, 0.0), (600, 0.04, 1.0), (24, 0.25, -0.7),
                                          (1024, 0.05, 0.5), (4096, 0.01, 0.0), (2048, 0.01, 0.3),
                                          (2048, 0.01, -0.7), (65536, 0.02, -2.0), (65536, 0.02, 1.2)])
def test_kernel_matches_reference(orc, ref, n, tau, drift):
    w_o, f_o, a_o, st = orc.kernel(n, tau, drift)
    assert st == 0
    w_r, f_r, a_r, st_r = ref.kernel(n, tau, drift)
    assert st_r == 0
    assert f_o == f_r and a_o == a_r
    assert np.array_equal(w_o, w_r)
    # the product's host builder (csrc/host/kernel_build.cpp) agrees too
    from paper_1210_4090_b200 import _capi
    import ctypes
    lib = _capi.load()
    w_p = np.empty(2 * n + 1)
    first, arg, delta = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    assert lib.lob_kernel_mech_host(None, n, tau, drift, w_p.ctypes.data, ctypes.byref(first),
                                    ctypes.byref(arg), ctypes.byref(delta)) == 0
    assert first.value == f_r and arg.value == a_r and np.array_equal(w_p, w_r)
    assert 0 < delta.value < 0.25


def test_kernel_kats(orc):
    # proj/tests/unit_scheme.cpp:45-58: P=0 symmetric, minimum 0 at the center
    w, first, arg, _ = orc.kernel(100, 0.1, 0.0)
    assert first == -100 and arg == 100 and w[100] == 0.0
    assert np.array_equal(w[:100][::-1], w[101:])
    # proj/tests/unit_scheme.cpp:60-67: N=600, tau=0.04, P=1 -> center 24, argmin 600
    w, first, arg, st = orc.kernel(600, 0.04, 1.0)
    assert first + 600 == 24 and arg == 600 and st == 0


# ---- min-plus KATs (proj/tests/unit_minplus.cpp) ------------------------------

def test_conv_naive_kats(orc, ref):
    assert list(orc.conv_naive([0.0, 1.0, 4.0], [0.0, 2.0])) == [0.0, 1.0, 3.0, 6.0]  # :111-116
    assert list(orc.conv_naive([0.0], [3.0, -1.0, 2.5, 0.0])) == [3.0, -1.0, 2.5, 0.0]  # :102-109
    r, _, _ = ref.conv(2, [4.0, 1.0, 0.0, 1.0, 4.0], [0.0, -1.0])  # :203-211
    assert list(r) == [4.0, 1.0, 0.0, -1.0, 0.0, 3.0]
    assert list(orc.conv_naive([4.0, 1.0, 0.0, 1.0, 4.0], [0.0, -1.0])) == list(r)
    r, _, _ = ref.conv(2, [4.0, 1.0, 0.0, 1.0, 4.0], [0.0, 2.0, 2.0, 0.0])  # :220-227
    assert list(r) == [4.0, 1.0, 0.0, 1.0, 1.0, 0.0, 1.0, 4.0]
    assert list(orc.conv_naive([4.0, 1.0, 0.0, 1.0, 4.0], [0.0, 2.0, 2.0, 0.0])) == list(r)


def test_conv_naive_random(orc, ref):
    rng = RNG(11)
    for _ in range(50):
        a, b = rng.uniform(-5, 5, 16), rng.uniform(-5, 5, 16)
        r, _, st = ref.conv(0, a, b)
        assert st == 0 and np.array_equal(orc.conv_naive(a, b), r)


# ---- decomposition (block counts) --------------------------------------------

def test_decompose_kats(orc, ref):
    v = np.cos(2.0 * 3.14159265358979 * np.arange(17) / 16.0)  # unit_minplus.cpp:283-292
    c, kinds, _, _ = ref.decompose(v)
    assert c == 3 and list(kinds) == [1, 0, 1]
    assert orc.decompose_count(v) == 3
    assert orc.decompose_count([3.0, 1.0, 0.0, 1.0, 3.0]) == 1
    assert orc.decompose_count([0.0, 1.0, 2.0, 3.0]) == 1
    w = 0.1 * np.arange(41) + np.where(np.arange(41) % 2 == 0, 1e-7, -1e-7)  # :307-315
    assert orc.decompose_count(w, 0.0) > 10 and orc.decompose_count(w, 1e-6) == 1
    assert orc.decompose_count([1.0, 5.0]) == 1 and orc.decompose_count([1.0]) == 1


@pytest.mark.parametrize("eta", [0.0, 1e-3, 0.5])
def test_decompose_counts_match_reference(orc, ref, eta):
    rng = RNG(19)
    for _ in range(200):
        v = rng.uniform(-1, 1, int(rng.integers(2, 200)))
        assert orc.decompose_count(v, eta) == ref.decompose(v, eta)[0]


# ---- periodic step: definition-level formula == kinetic_convolve ---------------

@pytest.mark.parametrize("drift", [0.0, 0.4, -0.7, 1.0])
def test_direct_equals_kinetic_convolve(orc, ref, drift):
    # proj/tests/unit_scheme.cpp:176-194 (N=24, tau=0.25) plus larger N
    rng = RNG(39)
    for n, tau in [(24, 0.25), (128, 0.125), (1024, 0.05)]:
        K, first, _, _ = orc.kernel(n, tau, drift)
        for _ in range(3):
            u = rand_periodic(rng, n)
            got = orc.direct(u[None, :], K, first)[0]
            for engine in (0, 1):  # Fast, Naive
                want, blocks, st = ref.kinetic_convolve(u, n, tau, drift, engine=engine)
                assert st == 0
                assert np.array_equal(got, want)
                assert blocks == orc.line_blocks(u)


def test_step_with_potential_matches_reference(orc, ref):
    rng = RNG(7)
    n, tau = 256, 0.05
    v = api.gen_potential(2, n)
    tv = api.tau_v(v, tau)
    drifts = np.array([-1.3, 0.0, 0.45, 2.0])
    u = rng.uniform(-1, 1, (4, n))
    want, blocks = ref.step_lines(u, tau, drifts, v=v, engine=1)
    for l, d in enumerate(drifts):
        K, first, _, _ = orc.kernel(n, tau, d)
        got = orc.direct(u[l:l + 1], K, first, tv=tv)[0]
        assert np.array_equal(got, want[l])


def test_windowed_matches_reference(orc, ref):
    rng = RNG(40)
    n, tau = 8, 0.25
    K, first, _, _ = orc.kernel(n, tau, 0.0)
    u = rng.uniform(-1, 1, 17)
    got, st = orc.window(u, n, K, first)
    want, _, st_r = ref.kinetic_convolve(u, n, tau, 0.0, engine=1, periodic=False)
    assert st == 0 and st_r == 0 and np.array_equal(got, want)


def test_split2d_matches_reference(orc, ref):
    # proj/tests/unit_splitting.cpp:103-121 and acceptance criterion 5
    rng = RNG(42)
    n, tau = 16, 0.25
    k1, f1, _, _ = orc.kernel(n, tau, 0.0)
    k2, f2, _, _ = orc.kernel(n, tau, 0.5)
    for _ in range(5):
        u = rng.uniform(-1, 1, (n, n))
        assert np.array_equal(orc.split2d(u, k1, f1, k2, f2), ref.split_step_2d(u, tau, 0.0, 0.5))


def test_split2d_c4_potential_matches_reference(orc, ref):
    n, tau, t = 32, 0.05, 0.35
    k1, f1, _, _ = orc.kernel(n, tau, 0.3)
    k2, f2, _, _ = orc.kernel(n, tau, -0.7)
    u = api.gen_c4_u0(n)
    a = api.gen_cos(n)
    b = api.c4_time_term(t + tau)
    v = np.add(np.multiply(a[:, None], a[None, :]), b)
    tv = api.tau_v(v, tau)
    got = orc.split2d(u, k1, f1, k2, f2, tv=tv)
    want = ref.split_step_2d(u, tau, 0.3, -0.7, pot_kind=1, t=t)
    assert np.array_equal(got, want)


def test_c1_evolve_drift_matches_reference(orc, ref):
    """Short C1 evolve: oracle stepping + sequential drift == reference evolve."""
    n, tau, steps = 1024, 0.05, 20
    u0 = api.gen_sin(n)
    v = api.gen_potential(1, n)
    tv = api.tau_v(v, tau)
    uf, drifts, blocks, comp = ref.evolve(u0, tau, 0.5, v, steps, engine=1)
    K, first, _, _ = orc.kernel(n, tau, 0.5)
    u = u0.copy()
    for i in range(steps):
        nxt = orc.direct(u[None, :], K, first, tv=tv)[0]
        d, fin = orc.drift(nxt, u)
        assert d == drifts[i] and fin
        assert orc.line_blocks(u) == blocks[i]
        u = nxt
    assert comp and np.array_equal(u, uf)
