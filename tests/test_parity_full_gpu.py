"""Parity at BASELINE.json's full sizes (SURVEY.md 8(d) "Parity gates"): C3 every line
against the reference itself, C4's first five split steps at 2048^2 against the
reference's split_step_nd, C5 sampled steps of the fast engine against the direct one,
C2's fast steps against the direct one on all 256 lines.  Every comparison is
bit-exact (==, +-0 equal)."""
import os

import numpy as np
import pytest

from paper_1210_4090_b200 import api

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def test_c3_every_line_vs_reference(dev, orc, ref):
    """C3: 4096 lines x N=4096, tau=0.01, P=0: K1 (screened and plain fp64) and K2 on every
    line == the reference's kinetic_convolve(..., ConvEngine::Naive) (oracle/_ref, all host
    threads); fp32 K1 == the fp32 restatement of the definition-level loop."""
    import torch
    n, tau, lines = 4096, 0.01, 4096
    u = api.gen_c3_lines(0, lines, n)
    want, _ = ref.step_lines(u, tau, 0.0, engine=0, nthreads=os.cpu_count() or 1, want_blocks=False)
    K = dev.build_kernel(n, tau, 0.0)
    du = to_dev(u)
    out = torch.empty_like(du)
    kt = to_dev(K.window)
    fr = torch.full((lines,), K.first, dtype=torch.int64, device="cuda")
    for mode in (api.DIRECT_SCREENED, api.DIRECT_PLAIN):
        dev.set_direct_mode(mode)
        dev.direct_f64(du, out, kt, fr)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), want), mode
    dev.set_direct_mode(api.DIRECT_SCREENED)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    dev.fast_f64(du, out, torch.zeros(lines, dtype=torch.float64, device="cuda"), tau, workspace=ws)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)
    c = dev.fast_counters(ws, lines, n)
    assert c["missed_outputs"] == 0 and c["direct_tiles_gate"] == 0 and c["direct_tiles_heavy"] == 0, c
    # fp32 (the reference has no fp32 path: the C restatement)
    u32 = u.astype(np.float32)
    k32 = K.window.astype(np.float32)
    o32 = torch.empty_like(to_dev(u32))
    dev.direct_f32(to_dev(u32), o32, to_dev(k32), fr)
    torch.cuda.synchronize()
    assert np.array_equal(o32.cpu().numpy(), orc.direct_f32(u32, k32, K.first, nthreads=os.cpu_count() or 1))


@pytest.mark.parametrize("engine,halves", [(api.ENGINE_FAST, 2), (api.ENGINE_FAST, 1), (api.ENGINE_DIRECT, 1)])
def test_c4_first_five_steps_vs_reference(dev, ref, engine, halves):
    """C4 at full size: 2048^2, tau=0.01, P=(0.3,-0.7), V=cos(2 pi x1)cos(2 pi x2)+0.2 sin(2 pi t)
    sampled at t+tau; steps 1..5 from u0 each == the reference's split_step_nd chain
    (proj/src/splitting.cpp:37-99)."""
    import torch
    n, tau = 2048, 0.01
    u = api.gen_c4_u0(n)
    a = to_dev(api.gen_cos(n))
    cur = to_dev(u)
    nxt, tmp = torch.empty_like(cur), torch.empty_like(cur)
    # two workspace halves: the fused four-launch step (one half per axis)
    ws = torch.empty(halves * dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
    ref_state = u
    for k in range(5):
        t = k * tau
        dev.split_step_2d(cur, nxt, tmp, tau, 0.3, -0.7, a1=a, a2=a, b=api.c4_time_term(t + tau),
                          engine=engine, workspace=ws)
        ref_state = ref.split_step_2d(ref_state, tau, 0.3, -0.7, pot_kind=1, t=t)
        torch.cuda.synchronize()
        assert np.array_equal(nxt.cpu().numpy(), ref_state), k + 1
        cur, nxt = nxt, cur


def test_c5_sampled_steps_fast_equals_direct(dev):
    """C5: 8 of the 64 lines (N=2^20, tau=0.005, P=0.25, V=0.5 sin(2 pi x)) stepped by the fast
    engine from u0; at steps 1, 100 and 199 the fast step == the direct step (K1, pinned to
    the reference) from the same state, every tile by the walk."""
    import torch
    n, tau = 1 << 20, 0.005
    idx = [0, 9, 18, 27, 36, 45, 54, 63]
    u0 = np.concatenate([api.gen_c5_lines(l, 1, n) for l in idx])
    lines = len(idx)
    cur = to_dev(u0)
    nxt = torch.empty_like(cur)
    tvn = api.tau_v(api.gen_potential(3, n), tau)
    tv = to_dev(tvn)
    dd = torch.full((lines,), 0.25, dtype=torch.float64, device="cuda")
    K = dev.build_kernel(n, tau, 0.25)
    kt = to_dev(K.window)
    fr = torch.full((lines,), K.first, dtype=torch.int64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    chk = torch.empty_like(cur)
    for step in range(1, 200):
        dev.fast_f64(cur, nxt, dd, tau, tv=tv, workspace=ws, flags=api.FAST_STATS_VALID if step > 1 else 0)
        if step in (1, 100, 199):
            dev.direct_f64(cur, chk, kt, fr, tv=tv)
            torch.cuda.synchronize()
            assert torch.equal(nxt, chk), step
        cur, nxt = nxt, cur
    c = dev.fast_counters(ws, lines, n)
    assert c["missed_outputs"] == 0 and c["direct_tiles_gate"] == 0 and c["direct_tiles_heavy"] == 0, c
