"""The resident evolve kernel (K2R: one CTA per short line, every step in one launch)
against the step-by-step K2 launch loop: final states and per-step block counts ==,
per-step drift <= 1e-12 (both device reductions; the reference's sequential sum is
pinned elsewhere)."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api

pytestmark = pytest.mark.gpu


def _evolve(dev, u0, drifts, tau, steps, tv, resident):
    import torch

    dev.set_evolve_resident(resident)
    try:
        u = torch.from_numpy(u0.copy()).cuda()
        scr = torch.empty_like(u)
        lines = u.shape[0]
        sd = torch.empty(steps * lines, dtype=torch.float64, device="cuda")
        sb = torch.empty(steps * lines, dtype=torch.int64, device="cuda")
        ws = torch.empty(dev.fast_workspace_bytes(lines, u.shape[1]), dtype=torch.uint8, device="cuda")
        done = dev.evolve(u, scr, torch.from_numpy(drifts).cuda(), tau, steps,
                          tv=None if tv is None else torch.from_numpy(tv).cuda(), step_drift=sd, step_blocks=sb,
                          workspace=ws)
        assert done == steps
        return u.cpu().numpy(), sd.cpu().numpy(), sb.cpu().numpy()
    finally:
        dev.set_evolve_resident(True)


@pytest.mark.parametrize("n,lines,steps,tau", [(64, 5, 300, 0.1), (1000, 3, 200, 0.05), (1024, 3, 200, 0.05),
                                               (4096, 2, 60, 0.02)])
def test_resident_evolve_equals_launch_loop(dev, n, lines, steps, tau):
    rng = np.random.default_rng(n)
    x = np.arange(n) / n
    u0 = np.stack([np.sin(2 * np.pi * x + rng.uniform(0, 6)) * rng.uniform(0.2, 1.0) for _ in range(lines)])
    drifts = np.linspace(-1.7, 1.9, lines)
    tv = api.tau_v(api.gen_potential(2, n), tau)
    a = _evolve(dev, u0, drifts, tau, steps, tv, True)
    b = _evolve(dev, u0, drifts, tau, steps, tv, False)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[2], b[2])
    assert np.max(np.abs(a[1] - b[1])) <= 1e-12


def test_evolve_loop_fused_drift(dev):
    """n > 4096 runs the step-by-step K2 loop with the drift's partial sums fused into the
    K2 epilogue: states == single K2 steps, drift <= 1e-12 of mean(u_next - u) per step"""
    import torch

    n, lines, steps, tau = 8192, 3, 12, 0.02
    rng = np.random.default_rng(3)
    x = np.arange(n) / n
    u0 = np.stack([np.sin(2 * np.pi * x + rng.uniform(0, 6)) for _ in range(lines)])
    drifts = np.array([0.3, -1.1, 1.7])
    tv = api.tau_v(api.gen_potential(2, n), tau)
    a = _evolve(dev, u0, drifts, tau, steps, tv, True)
    u = torch.from_numpy(u0.copy()).cuda()
    out = torch.empty_like(u)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    dr = torch.from_numpy(drifts).cuda()
    dtv = torch.from_numpy(tv).cuda()
    bl = torch.empty(lines, dtype=torch.int64, device="cuda")
    for k in range(steps):
        dev.fast_f64(u, out, dr, tau, tv=dtv, blocks=bl, workspace=ws, flags=api.FAST_STATS_VALID if k else 0)
        want = (out - u).mean(dim=1).cpu().numpy()
        assert np.max(np.abs(a[1][k * lines:(k + 1) * lines] - want)) <= 1e-12
        assert np.array_equal(a[2][k * lines:(k + 1) * lines], bl.cpu().numpy())
        u, out = out, u
    assert np.array_equal(a[0], u.cpu().numpy())


def test_k2_block_counts_after_steps_without_them(dev, orc):
    """K2 skips decompose()'s FSM when a call asks for no block counts; a later call that does
    ask recomputes the statistics: outputs and counts stay exact in any interleaving."""
    import torch

    n, lines, tau = 4096, 3, 0.02
    rng = np.random.default_rng(8)
    u = np.cumsum(rng.uniform(-1.0 / n, 1.0 / n, (lines, n)), axis=1)
    u -= np.linspace(0, 1, n)[None, :] * u[:, -1:]
    drifts = np.array([0.2, -0.9, 1.4])
    a = torch.from_numpy(u).cuda()
    b = torch.empty_like(a)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    dr = torch.from_numpy(drifts).cuda()
    bl = torch.empty(lines, dtype=torch.int64, device="cuda")
    pattern = [True, False, False, True, True, False, True]
    for k, want_blocks in enumerate(pattern):
        x = a.cpu().numpy()
        dev.fast_f64(a, b, dr, tau, blocks=bl if want_blocks else None, workspace=ws,
                     flags=api.FAST_STATS_VALID if k else 0)
        y = b.cpu().numpy()
        for l in range(lines):
            w, first, _, _ = orc.kernel(n, tau, drifts[l])
            assert np.array_equal(y[l], orc.direct(x[l:l + 1], w, first)[0])
            if want_blocks:
                assert bl[l].item() == orc.line_blocks(x[l])
        a, b = b, a


@pytest.mark.parametrize("n,tau", [(64, 0.1), (1000, 0.03), (4096, 0.01)])
def test_resident_structured_inputs(dev, n, tau):
    """K2R on the adversarial shapes of tests/test_fast_gpu.py (constant, exact ties, jumps,
    1e8 magnitudes, spikes, near-ties) == the K2 launch loop: states and block counts."""
    from tests.test_fast_gpu import _structured_lines

    u0 = _structured_lines(n, np.random.default_rng(n))
    drifts = np.linspace(-0.9, 1.3, u0.shape[0])
    a = _evolve(dev, u0, drifts, tau, 25, None, True)
    b = _evolve(dev, u0, drifts, tau, 25, None, False)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[2], b[2])
    assert np.max(np.abs(a[1] - b[1])) <= 1e-12 * max(1.0, float(np.max(np.abs(u0))))
