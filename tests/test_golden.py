"""Golden vectors produced by the reference itself (tests/golden/make_golden.py,
run where /root/reference is present).  CPU tests pin the C oracle and the
product's host kernel builder to them; GPU tests pin K1/K2/K3."""
import os

import numpy as np
import pytest

from paper_1210_4090_b200 import api

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(G, name))


# ---------------------------------------------------------------- CPU (oracle pin)

def test_oracle_kernels_match_golden(orc):
    g = load("kernels.npz")
    for key in g.files:
        if not key.startswith("w_"):
            continue
        _, n, tau, p = key.split("_")
        w, first, arg, _ = orc.kernel(int(n), float(tau), float(p))
        meta = g["meta_" + key[2:]]
        assert np.array_equal(w, g[key]) and first == meta[0] and arg == meta[1], key


def test_product_kernel_builder_matches_golden():
    import ctypes
    from paper_1210_4090_b200 import _capi
    lib = _capi.load()
    g = load("kernels.npz")
    for key in g.files:
        if not key.startswith("w_"):
            continue
        _, n, tau, p = key.split("_")
        w = np.empty(2 * int(n) + 1)
        first, arg, delta = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
        assert lib.lob_kernel_mech_host(None, int(n), float(tau), float(p), w.ctypes.data, ctypes.byref(first),
                                        ctypes.byref(arg), ctypes.byref(delta)) == 0
        assert np.array_equal(w, g[key]) and first.value == g["meta_" + key[2:]][0]


def test_oracle_kinetic_convolve_golden(orc):
    g = load("kinetic_convolve_n24.npz")
    for drift in (0.0, 0.4, -0.7, 1.0):
        w, first, _, _ = orc.kernel(24, 0.25, drift)
        u = g[f"u_{drift}"]
        assert np.array_equal(orc.direct(u[None, :], w, first)[0], g[f"out_{drift}"])
        assert orc.line_blocks(u) == g[f"blocks_{drift}"][0]


def test_oracle_c1_full_evolve_golden(orc):
    """C1 in full (2000 steps) with the oracle: final state, per-step drift and
    block counts == the reference's evolve; H-bar = -1.0074376402935734."""
    g = load("c1_evolve.npz")
    n, tau = 1024, 0.05
    w, first, _, _ = orc.kernel(n, tau, 0.5)
    tv = api.tau_v(g["v"], tau)
    u = g["u0"].copy()
    for i in range(2000):
        nxt = orc.direct(u[None, :], w, first, tv=tv)[0]
        d, fin = orc.drift(nxt, u)
        assert d == g["step_drift"][i] and fin
        if i % 97 == 0:
            assert orc.line_blocks(u) == g["step_blocks"][i]
        u = nxt
    assert np.array_equal(u, g["u_final"])
    hbar = np.sum(u - g["u0"]) / n / (2000 * tau)
    assert hbar == g["hbar"][0]
    assert abs(hbar - (-1.007437640293573)) < 1e-15  # SURVEY.md section 8c measured value


def test_oracle_c3_c2_split_decompose_golden(orc):
    g = load("c3_lines0-3.npz")
    w, first, _, _ = orc.kernel(4096, 0.01, 0.0)
    assert np.array_equal(orc.direct(g["u"], w, first), g["out"])
    assert [orc.line_blocks(x) for x in g["u"]] == list(g["blocks"])
    g = load("c2_n2048_5steps.npz")
    tv = api.tau_v(g["v"], 0.02)
    u = np.zeros((4, 2048))
    for s in range(5):
        u = np.stack([orc.direct(u[l:l + 1], *orc.kernel(2048, 0.02, d)[:2], tv=tv)[0]
                      for l, d in enumerate(g["drifts"])])
        assert np.array_equal(u, g["states"][s])
    g = load("split2d.npz")
    k1, f1, _, _ = orc.kernel(16, 0.25, 0.0)
    k2, f2, _, _ = orc.kernel(16, 0.25, 0.5)
    assert np.array_equal(orc.split2d(g["u16"], k1, f1, k2, f2), g["out16"])
    g = load("decompose.npz")
    off = 0
    for L, c in zip(g["lens"], g["counts"]):
        x = g["values"][off:off + L]
        off += L
        assert [orc.decompose_count(x, eta) for eta in (0.0, 1e-3, 0.5)] == list(c)


# ---------------------------------------------------------------- GPU

def to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.gpu
@pytest.mark.parametrize("engine", [api.ENGINE_FAST, api.ENGINE_DIRECT])
def test_gpu_c1_full_evolve_golden(dev, engine):
    import torch
    g = load("c1_evolve.npz")
    n, tau, steps = 1024, 0.05, 2000
    u = to_dev(g["u0"][None, :])
    scratch = torch.empty_like(u)
    sd = torch.empty(steps, dtype=torch.float64, device="cuda")
    sb = torch.empty(steps, dtype=torch.int64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(1, n), dtype=torch.uint8, device="cuda")
    done = dev.evolve(u, scratch, to_dev(np.array([0.5])), tau, steps, tv=to_dev(api.tau_v(g["v"], tau)),
                      engine=engine, step_drift=sd, step_blocks=sb, workspace=ws)
    assert done == steps
    uf = u.cpu().numpy()[0]
    assert np.array_equal(uf, g["u_final"])
    assert np.array_equal(sb.cpu().numpy(), g["step_blocks"])
    assert np.max(np.abs(sd.cpu().numpy() - g["step_drift"])) <= 1e-12
    hbar = np.sum(uf - g["u0"]) / n / (steps * tau)
    assert abs(hbar - g["hbar"][0]) <= 1e-12 * abs(g["hbar"][0])


@pytest.mark.gpu
def test_gpu_c3_c2_split_golden(dev):
    import torch
    g = load("c3_lines0-3.npz")
    out = torch.empty((4, 4096), dtype=torch.float64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(4, 4096), dtype=torch.uint8, device="cuda")
    blocks = torch.empty(4, dtype=torch.int64, device="cuda")
    dev.fast_f64(to_dev(g["u"]), out, to_dev(np.zeros(4)), 0.01, blocks=blocks, workspace=ws)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), g["out"])
    assert list(blocks.cpu().numpy()) == list(g["blocks"])
    g = load("c2_n2048_5steps.npz")
    u = torch.zeros((4, 2048), dtype=torch.float64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(4, 2048), dtype=torch.uint8, device="cuda")
    dd, dtv = to_dev(g["drifts"]), to_dev(api.tau_v(g["v"], 0.02))
    for s in range(5):
        nxt = torch.empty_like(u)
        dev.fast_f64(u, nxt, dd, 0.02, tv=dtv, workspace=ws, flags=api.FAST_STATS_VALID if s else 0)
        u = nxt
        torch.cuda.synchronize()
        assert np.array_equal(u.cpu().numpy(), g["states"][s])
    g = load("split2d.npz")
    for engine in (api.ENGINE_DIRECT, api.ENGINE_FAST):
        du = to_dev(g["u16"])
        o, t = torch.empty_like(du), torch.empty_like(du)
        wsp = torch.empty(dev.fast_workspace_bytes(16, 16), dtype=torch.uint8, device="cuda")
        dev.split_step_2d(du, o, t, 0.25, 0.0, 0.5, engine=engine, workspace=wsp)
        torch.cuda.synchronize()
        assert np.array_equal(o.cpu().numpy(), g["out16"])
        a = api.gen_cos(32)
        du = to_dev(g["u32"])
        o, t = torch.empty_like(du), torch.empty_like(du)
        wsp = torch.empty(dev.fast_workspace_bytes(32, 32), dtype=torch.uint8, device="cuda")
        dev.split_step_2d(du, o, t, 0.05, 0.3, -0.7, a1=to_dev(a), a2=to_dev(a),
                          b=api.c4_time_term(0.35 + 0.05), engine=engine, workspace=wsp)
        torch.cuda.synchronize()
        assert np.array_equal(o.cpu().numpy(), g["out32"])


# ---------------------------------------------------------------- long-run fixtures (make_golden_long.py)

def test_oracle_c2_hbar_sweep_n1024_golden(orc):
    """One line of the N=1024 C2 sweep in full (5000 steps) with the oracle."""
    g = load("c2_hbar_n1024.npz")
    n, tau, k = 1024, 0.02, 1  # keep[1] = line 37
    line = int(g["keep"][k])
    w, first, _, _ = orc.kernel(n, tau, float(g["drifts"][line]))
    tv = api.tau_v(g["v"], tau)
    u = np.zeros(n)
    for i in range(5000):
        nxt = orc.direct(u[None, :], w, first, tv=tv)[0]
        if i % 499 == 0:
            assert orc.drift(nxt, u)[0] == g["step_drift"][k][i]
        u = nxt
    assert np.array_equal(u, g["u_final"][k])
    assert np.sum(u) / n / (5000 * tau) == g["hbar"][line]


def test_oracle_c4_n128_golden(orc):
    g = load("c4_n128.npz")
    n, tau = 128, 0.01
    k1, f1, _, _ = orc.kernel(n, tau, 0.3)
    k2, f2, _, _ = orc.kernel(n, tau, -0.7)
    a = api.gen_cos(n)
    u, k = g["u0"], 0
    for i in range(int(g["at"][-1]) + 1):
        tv = api.tau_v(np.add.outer(a, np.zeros(n)) * a[None, :] + api.c4_time_term(i * tau + tau), tau)
        u = orc.split2d(u, k1, f1, k2, f2, tv=tv)
        if i == g["at"][k]:
            assert np.array_equal(u, g["states"][k]), i
            k += 1


@pytest.mark.gpu
def test_gpu_c2_hbar_sweep_n1024_golden(dev):
    """All 256 C2 drifts, 5000 steps at N=1024 (K2 via lob_evolve_f64): H-bar(P)
    within 1e-12 relative of the reference's, kept lines bit-exact."""
    import torch
    g = load("c2_hbar_n1024.npz")
    n, tau, steps, lines = 1024, 0.02, 5000, 256
    u = torch.zeros((lines, n), dtype=torch.float64, device="cuda")
    sc = torch.empty_like(u)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    sb = torch.empty((steps, lines), dtype=torch.int64, device="cuda")
    sd = torch.empty((steps, lines), dtype=torch.float64, device="cuda")
    assert dev.evolve(u, sc, to_dev(g["drifts"]), tau, steps, tv=to_dev(api.tau_v(g["v"], tau)),
                      step_drift=sd, step_blocks=sb, workspace=ws) == steps
    uf = u.cpu().numpy()
    hb = uf.sum(axis=1) / n / (steps * tau)
    assert np.max(np.abs(hb - g["hbar"]) / np.abs(g["hbar"])) <= 1e-12
    assert np.array_equal(uf[g["keep"]], g["u_final"])
    assert np.array_equal(sb.cpu().numpy()[:, g["keep"]].T, g["step_blocks"])
    assert np.max(np.abs(sd.cpu().numpy()[:, g["keep"]].T - g["step_drift"])) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("engine", [api.ENGINE_FAST, api.ENGINE_DIRECT])
def test_gpu_c5_spectrum_n16384_golden(dev, engine):
    import torch
    g = load("c5_n16384.npz")
    n, tau, steps = 1 << 14, 0.005, 40
    u = to_dev(g["u0"])
    sc = torch.empty_like(u)
    ws = torch.empty(dev.fast_workspace_bytes(2, n), dtype=torch.uint8, device="cuda")
    sb = torch.empty((steps, 2), dtype=torch.int64, device="cuda")
    assert dev.evolve(u, sc, to_dev(np.full(2, 0.25)), tau, steps, tv=to_dev(api.tau_v(g["v"], tau)),
                      engine=engine, step_blocks=sb, workspace=ws) == steps
    assert np.array_equal(u.cpu().numpy(), g["u_final"])
    assert np.array_equal(sb.cpu().numpy().T, g["step_blocks"])


@pytest.mark.gpu
@pytest.mark.parametrize("engine", [api.ENGINE_FAST, api.ENGINE_DIRECT])
def test_gpu_c4_n128_golden(dev, engine):
    import torch
    g = load("c4_n128.npz")
    n, tau = 128, 0.01
    a = to_dev(api.gen_cos(n))
    u = to_dev(g["u0"])
    o, t = torch.empty_like(u), torch.empty_like(u)
    ws = torch.empty(dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
    k = 0
    for i in range(int(g["at"][-1]) + 1):
        dev.split_step_2d(u, o, t, tau, 0.3, -0.7, a1=a, a2=a, b=api.c4_time_term(i * tau + tau),
                          engine=engine, workspace=ws)
        u, o = o, u
        if i == g["at"][k]:
            torch.cuda.synchronize()
            assert np.array_equal(u.cpu().numpy(), g["states"][k]), i
            k += 1
