"""K2 over the reference's kernel WINDOW (lob_minplus_fast_window_f64): the fast exact engine
for any convex window — mechanical or tabulated (proj/src/hamiltonian.cpp:30-82,
proj/src/scheme.cpp:59-105) — i.e. what kinetic_convolve(u, kernel, eta, engine, blocks)
hands an engine (proj/include/laxol/scheme.hpp:52-53).  Bit-exact against the reference /
the oracle's direct formula, and the walk (not the direct fallback) is asserted to run."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api
from tests.test_fast_gpu import assert_walk, oracle_step, rough_walk, to_dev
from tests.test_tabulated import TABLES, table

pytestmark = pytest.mark.gpu


def window_step(dev, u, K, first, tau, tv=None, ws=None, flags=0, blocks=False):
    import torch
    lines, n = u.shape
    du = to_dev(u) if isinstance(u, np.ndarray) else u
    out = torch.empty_like(du)
    if ws is None:
        ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    K = np.atleast_2d(K)
    kt = to_dev(K)
    fr = to_dev(np.broadcast_to(np.asarray(first, np.int64), (lines,)).copy())
    bl = torch.empty(lines, dtype=torch.int64, device="cuda") if blocks else None
    dev.fast_window_f64(du, out, kt, fr, tau, tv=None if tv is None else to_dev(tv), workspace=ws, flags=flags,
                        ktab_stride=0 if K.shape[0] == 1 else K.shape[1], blocks=bl)
    torch.cuda.synchronize()
    return out, ws, (bl.cpu().numpy() if blocks else None)


@pytest.mark.parametrize("drift", [0.0, 0.4, -0.7])
@pytest.mark.parametrize("n,tau", [(48, 0.125), (600, 0.04), (1024, 0.05), (4096, 0.01)])
def test_window_mechanical_equals_oracle_and_drift_engine(dev, orc, n, tau, drift):
    rng = np.random.default_rng(n + 3)
    u = rough_walk(rng, 4, n, 4.0)
    K, first, _, _ = orc.kernel(n, tau, drift)
    got, ws, blocks = window_step(dev, u, K, first, tau, blocks=True)
    assert np.array_equal(got.cpu().numpy(), oracle_step(orc, u, drift, tau))
    assert [orc.line_blocks(u[l]) for l in range(4)] == list(blocks)
    assert_walk(dev.fast_counters(ws, 4, n))


@pytest.mark.parametrize("name", list(TABLES))
@pytest.mark.parametrize("n,tau", [(64, 0.05), (256, 0.1), (1024, 0.02)])
def test_window_tabulated_equals_reference(dev, ref, name, n, tau):
    s, v0, dv = table(name)
    K, first, _, st = ref.kernel_tabulated(n, tau, s, v0, dv)
    if st != 0:
        pytest.skip("the reference rejects this window")
    rng = np.random.default_rng(len(name) + n)
    u = rng.uniform(-0.05, 0.05, (3, n)).cumsum(axis=1)
    u -= np.linspace(0, 1, n)[None, :] * u[:, -1:]
    got, ws, _ = window_step(dev, u, K, first, tau)
    g = got.cpu().numpy()
    for l in range(3):
        want, _, st = ref.convolve_tabulated(u[l], tau, s, v0, dv, 0.0, engine=1)
        assert st == 0 and np.array_equal(g[l], want), l
    c = dev.fast_counters(ws, 3, n)
    assert c["missed_outputs"] == 0 and c["tiles"] > 0, c


def test_window_per_line_tables_c2_slice_equals_direct(dev):
    """C2-like lines (N=65536, per-line mechanical windows, potential) stepped 40 times by the
    window engine with carried statistics; the last step == K1 on every line, all walk."""
    import torch
    n, tau = 65536, 0.02
    drifts = api.gen_c2_drifts(256)[[0, 60, 128, 200, 255]]
    ks = [dev.build_kernel(n, tau, float(p)) for p in drifts]
    K = np.stack([k.window for k in ks])
    first = np.array([k.first for k in ks], np.int64)
    tv = to_dev(api.tau_v(api.gen_potential(2, n), tau))
    lines = len(drifts)
    u = torch.zeros((lines, n), dtype=torch.float64, device="cuda")
    v = torch.empty_like(u)
    kt, fr = to_dev(K), to_dev(first)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    for i in range(40):
        dev.fast_window_f64(u, v, kt, fr, tau, tv=tv, workspace=ws, ktab_stride=2 * n + 1,
                            flags=api.FAST_STATS_VALID if i else 0)
        u, v = v, u
    ws2 = torch.empty_like(ws)
    dev.fast_window_f64(u, v, kt, fr, tau, tv=tv, workspace=ws2, ktab_stride=2 * n + 1)
    w = torch.empty_like(u)
    dev.direct_f64(u, w, kt, fr, tv=tv, ktab_stride=2 * n + 1)
    torch.cuda.synchronize()
    assert torch.equal(v, w)
    assert_walk(dev.fast_counters(ws2, lines, n))


def test_window_table_change_recomputes_statistics(dev, orc):
    """Carried statistics belong to the table they were computed with: a call with another
    window but LOB_FAST_STATS_VALID recomputes the line constants (still exact)."""
    import torch
    n, tau = 1024, 0.05
    rng = np.random.default_rng(5)
    u = rough_walk(rng, 2, n, 3.0)
    K1, f1, _, _ = orc.kernel(n, tau, 0.3)
    K2, f2, _, _ = orc.kernel(n, tau, -0.9)
    a, ws, _ = window_step(dev, u, K1, f1, tau)
    b, _, _ = window_step(dev, a, K2, f2, tau, ws=ws, flags=api.FAST_STATS_VALID)
    assert np.array_equal(b.cpu().numpy(), oracle_step(orc, a.cpu().numpy(), -0.9, tau))
    # the same with the second window written over the first one's device buffer (one address)
    import torch
    kt = to_dev(K1)
    fr = to_dev(np.full(2, f1, np.int64))
    ws = torch.empty(dev.fast_workspace_bytes(2, n), dtype=torch.uint8, device="cuda")
    du = to_dev(u)
    x, y = torch.empty_like(du), torch.empty_like(du)
    dev.fast_window_f64(du, x, kt, fr, tau, workspace=ws)
    kt.copy_(to_dev(K2))
    fr.fill_(f2)
    dev.fast_window_f64(x, y, kt, fr, tau, workspace=ws, flags=api.FAST_STATS_VALID)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), oracle_step(orc, x.cpu().numpy(), -0.9, tau))
    assert dev.fast_counters(ws, 2, n)["stale_line_constants"] > 0


@pytest.mark.parametrize("line_kernel", [False, True])
def test_drift_changed_in_place_is_detected(dev, orc, line_kernel):
    """lob_minplus_fast_f64 with carried statistics after the drift array was rewritten in place:
    the tiles see the mismatch, take the direct formula with the current drift (exact), counted.
    The whole-line kernel (K2L, n <= 2048) carries nothing: it reads the current drift."""
    import torch
    n, tau = 2048, 0.02
    rng = np.random.default_rng(9)
    du = to_dev(rough_walk(rng, 3, n, 3.0))
    dd = to_dev(np.full(3, 0.2))
    x, y = torch.empty_like(du), torch.empty_like(du)
    ws = torch.empty(dev.fast_workspace_bytes(3, n), dtype=torch.uint8, device="cuda")
    dev.set_fast_line(line_kernel)
    try:
        dev.fast_f64(du, x, dd, tau, workspace=ws)
        dd.fill_(-1.3)
        dev.fast_f64(x, y, dd, tau, workspace=ws, flags=api.FAST_STATS_VALID)
        torch.cuda.synchronize()
    finally:
        dev.set_fast_line(2)
    assert np.array_equal(y.cpu().numpy(), oracle_step(orc, x.cpu().numpy(), -1.3, tau))
    c = dev.fast_counters(ws, 3, n)
    if line_kernel:
        assert c["stale_line_constants"] == 0 and c["missed_outputs"] == 0, c
    else:
        assert c["stale_line_constants"] > 0, c
