"""Device-resident evolve (lob_evolve_f64): per-step drift, block counts and
the non-finite abort (proj/src/scheme.cpp:208-272), against the reference."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api

pytestmark = pytest.mark.gpu


def to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("engine", [api.ENGINE_FAST, api.ENGINE_DIRECT])
def test_evolve_batch_matches_reference_per_line(dev, ref, engine):
    """8 C2-like lines at N=1024 (P over [-2, 2]), 200 steps: final states
    bit-identical to the reference's evolve, drifts within 1e-12, block counts equal."""
    import torch
    n, tau, steps = 1024, 0.02, 200
    drifts = api.gen_c2_drifts(256)[::32]
    v = api.gen_potential(2, n)
    tv = api.tau_v(v, tau)
    lines = len(drifts)
    u = torch.zeros((lines, n), dtype=torch.float64, device="cuda")
    scratch = torch.empty_like(u)
    sd = torch.empty((steps, lines), dtype=torch.float64, device="cuda")
    sb = torch.empty((steps, lines), dtype=torch.int64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    done = dev.evolve(u, scratch, to_dev(drifts), tau, steps, tv=to_dev(tv), engine=engine,
                      step_drift=sd, step_blocks=sb, workspace=ws)
    assert done == steps
    got = u.cpu().numpy()
    for l, d in enumerate(drifts):
        uf, dr, bl, comp = ref.evolve(np.zeros(n), tau, float(d), v, steps, engine=1)
        assert comp
        assert np.array_equal(got[l], uf)
        assert np.max(np.abs(sd.cpu().numpy()[:, l] - dr)) <= 1e-12
        assert np.array_equal(sb.cpu().numpy()[:, l], bl)


def test_evolve_abort_on_nonfinite(dev):
    """A potential that overflows u to -inf stops the device loop and reports
    the step (EvaluationError, like EvolutionTrace.completed = false)."""
    import torch
    n, tau = 64, 0.25
    u = torch.zeros((1, n), dtype=torch.float64, device="cuda")
    scratch = torch.empty_like(u)
    tv = to_dev(np.full(n, tau * 1e308))
    ws = torch.empty(dev.fast_workspace_bytes(1, n), dtype=torch.uint8, device="cuda")
    with pytest.raises(api.EvaluationError):
        dev.evolve(u, scratch, to_dev(np.zeros(1)), tau, 40, tv=tv, workspace=ws)


def test_step_host_e2e_matches_device(dev, orc):
    """The host-buffer entry (lob_step_host_f64, the e2e path) == the oracle."""
    n, tau = 4096, 0.02
    drifts = np.array([-1.5, 0.25, 1.75])
    tv = api.tau_v(api.gen_potential(2, n), tau)
    rng = np.random.default_rng(3)
    u = np.cumsum(rng.uniform(-1.0 / n, 1.0 / n, (3, n)), axis=1)
    u -= np.linspace(0, 1, n, endpoint=False)[None, :] * u[:, -1:]
    blocks = np.empty(3, np.int64)
    for engine in (api.ENGINE_FAST, api.ENGINE_DIRECT):
        out = dev.step_host(u, drifts, tau, tv=tv, engine=engine, blocks=blocks)
        for l, d in enumerate(drifts):
            K, first, _, _ = orc.kernel(n, tau, d)
            assert np.array_equal(out[l], orc.direct(u[l:l + 1], K, first, tv=tv)[0])
            assert blocks[l] == orc.line_blocks(u[l])


@pytest.mark.parametrize("per_line_tv", [False, True])
def test_step_host_pipelined_chunks_match_device(dev, per_line_tv):
    """>= 16 lines take the two-stream chunked host path (uneven last chunk):
    same doubles and block counts as one device-resident K2 call."""
    import torch
    n, tau, lines = 2048, 0.02, 37
    drifts = api.gen_c2_drifts(256)[:lines * 6:6].copy()
    rng = np.random.default_rng(11)
    u = np.cumsum(rng.uniform(-1.0 / n, 1.0 / n, (lines, n)), axis=1)
    u -= np.linspace(0, 1, n, endpoint=False)[None, :] * u[:, -1:]
    v = api.gen_potential(2, n)
    tv = api.tau_v(np.stack([v * (1 + 0.01 * l) for l in range(lines)]) if per_line_tv else v, tau)
    stride = n if per_line_tv else 0
    blocks = np.empty(lines, np.int64)
    out = dev.step_host(u, drifts, tau, tv=tv, tv_stride=stride, blocks=blocks)
    du, dout = to_dev(u), torch.empty((lines, n), dtype=torch.float64, device="cuda")
    db = torch.empty(lines, dtype=torch.int64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    dev.fast_f64(du, dout, to_dev(drifts), tau, tv=to_dev(tv), tv_stride=stride, blocks=db, workspace=ws)
    torch.cuda.synchronize()
    assert np.array_equal(out, dout.cpu().numpy())
    assert np.array_equal(blocks, db.cpu().numpy())
