"""Edge cases of the stepping path through the C-ABI, against the reference itself:
empty batches, zero steps, the smallest grids the reference accepts (n_space = 1, 2, ...,
proj/src/scheme.cpp:40), grids one sample either side of the K2 tile and K2L limits, and
the argument checks that map to the reference's InvalidInput (proj/src/scheme.cpp:39-53)."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api

pytestmark = pytest.mark.gpu


def to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def windows(dev, n, tau, drifts):
    import torch
    ks = [dev.build_kernel(n, tau, float(d)) for d in drifts]
    kt = to_dev(np.concatenate([k.window for k in ks]))
    fr = torch.tensor([k.first for k in ks], dtype=torch.int64, device="cuda")
    return kt, fr


def all_engines(dev, u, drifts, tau, tv=None):
    """One step of the same lines through K1 (screened and plain), K2, the window-table K2 and
    the relaxed engine at eta = 0; returns {name: ndarray}."""
    import torch
    lines, n = u.shape
    du, dd = to_dev(u), to_dev(drifts)
    dtv = None if tv is None else to_dev(tv)
    kt, fr = windows(dev, n, tau, drifts)
    res = {}
    for name, mode in (("k1_screened", api.DIRECT_SCREENED), ("k1_plain", api.DIRECT_PLAIN)):
        dev.set_direct_mode(mode)
        o = torch.empty_like(du)
        dev.direct_f64(du, o, kt, fr, tv=dtv, ktab_stride=2 * n + 1)
        res[name] = o
    dev.set_direct_mode(api.DIRECT_SCREENED)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    o = torch.empty_like(du)
    dev.fast_f64(du, o, dd, tau, tv=dtv, workspace=ws)
    res["k2"] = o
    o = torch.empty_like(du)
    ws2 = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    dev.fast_window_f64(du, o, kt, fr, tau, tv=dtv, workspace=ws2, ktab_stride=2 * n + 1)
    res["k2_window"] = o
    o = torch.empty_like(du)
    dev.relaxed_f64(du, o, kt, fr, 0.0, tv=dtv, ktab_stride=2 * n + 1)
    res["relaxed_eta0"] = o
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in res.items()}


@pytest.mark.parametrize("n", [1, 2, 3, 4, 6])
def test_smallest_grids_equal_the_reference(dev, ref, n):
    """n_space = 1 is legal in the reference (SchemeParams: n_space >= 1); every engine gives
    the reference's step on the smallest periodic grids (the window spans two periods of a line
    shorter than a warp)."""
    tau, lines = 1.5, 5  # epsilon/tau = 1/(1.5 n) < 1
    rng = np.random.default_rng(n)
    u = rng.uniform(-1, 1, (lines, n))
    drifts = np.array([0.0, 0.4, -0.7, 1.0, -2.5])
    v = rng.uniform(-1, 1, n)
    want, _ = ref.step_lines(u, tau, drifts, v=v, engine=1)
    for name, got in all_engines(dev, u, drifts, tau, tv=tau * v).items():
        assert np.array_equal(got, want), (name, n)


@pytest.mark.parametrize("n", [2047, 2048, 2049, 2050, 4095, 4097])
def test_grids_around_the_tile_and_line_kernel_limits(dev, ref, n):
    """One sample either side of K2L's whole-line limit and K2's 2048-output tile (a last tile of
    1 or 2 outputs), odd and even: == the reference's step (Naive engine) for K1 and K2."""
    import torch
    tau, lines = 0.01, 3
    rng = np.random.default_rng(n)
    u = np.cumsum(rng.uniform(-1.0 / n, 1.0 / n, (lines, n)), axis=1)
    u -= np.linspace(0, 1, n, endpoint=False)[None, :] * u[:, -1:]
    u += 0.2 * np.sin(2 * np.pi * np.arange(n) / n)[None, :]
    drifts = np.array([0.3, -0.7, 1.9])
    want, wb = ref.step_lines(u, tau, drifts, engine=1, nthreads=3)
    du, dd = to_dev(u), to_dev(drifts)
    kt, fr = windows(dev, n, tau, drifts)
    o1 = torch.empty_like(du)
    dev.direct_f64(du, o1, kt, fr, ktab_stride=2 * n + 1)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    o2 = torch.empty_like(du)
    bl = torch.empty(lines, dtype=torch.int64, device="cuda")
    dev.fast_f64(du, o2, dd, tau, blocks=bl, workspace=ws)
    torch.cuda.synchronize()
    assert np.array_equal(o1.cpu().numpy(), want)
    assert np.array_equal(o2.cpu().numpy(), want)
    assert list(bl.cpu().numpy()) == list(wb)
    c = dev.fast_counters(ws, lines, n)
    assert c["missed_outputs"] == 0, c


def test_empty_batch_is_a_no_op(dev):
    """lines = 0: every batched entry returns success without touching anything."""
    import torch
    n, tau = 64, 0.05
    u = torch.empty((0, n), dtype=torch.float64, device="cuda")
    out = torch.empty_like(u)
    dd = torch.empty(0, dtype=torch.float64, device="cuda")
    k = dev.build_kernel(n, tau, 0.5)
    kt = to_dev(k.window)
    fr = torch.tensor([k.first], dtype=torch.int64, device="cuda")
    ws = torch.empty(max(1, dev.fast_workspace_bytes(1, n)), dtype=torch.uint8, device="cuda")
    dev.direct_f64(u, out, kt, fr)
    dev.fast_f64(u, out, dd, tau, workspace=ws)
    dev.fast_window_f64(u, out, kt, fr, tau, workspace=ws)
    dev.relaxed_f64(u, out, kt, fr, 0.0, workspace=ws)
    assert dev.evolve(u, out, dd, tau, 3, workspace=ws) in (0, 3)
    got = dev.step_host(np.empty((0, n)), np.empty(0), tau)
    assert got.shape == (0, n)
    torch.cuda.synchronize()


def test_zero_steps_leave_the_state_untouched(dev):
    import torch
    n, tau, lines = 256, 0.05, 2
    rng = np.random.default_rng(1)
    u = rng.uniform(-1, 1, (lines, n))
    du = to_dev(u)
    sc = torch.full_like(du, 7.0)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    for eng in (api.ENGINE_FAST, api.ENGINE_DIRECT):
        done = dev.evolve(du, sc, to_dev(np.array([0.5, -0.5])), tau, 0, engine=eng, workspace=ws)
        torch.cuda.synchronize()
        assert done == 0
        assert np.array_equal(du.cpu().numpy(), u)


def test_invalid_arguments_map_to_invalid_input(dev):
    """The reference's validate(SchemeParams) (proj/src/scheme.cpp:39-53): n_space < 1, tau <= 0,
    eta < 0 and the anti-CFL bound epsilon/tau >= h0 = 1 all throw InvalidInput; so do the
    C-ABI entries, before any launch."""
    import torch
    n = 64
    u = torch.zeros((2, n), dtype=torch.float64, device="cuda")
    out = torch.empty_like(u)
    dd = torch.zeros(2, dtype=torch.float64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(2, n), dtype=torch.uint8, device="cuda")
    with pytest.raises(api.InvalidInput):
        dev.fast_f64(u, out, dd, 0.0, workspace=ws)  # tau must be positive
    with pytest.raises(api.InvalidInput):
        dev.fast_f64(u, out, dd, -0.1, workspace=ws)
    with pytest.raises(api.InvalidInput):
        dev.fast_f64(u, out, dd, 1.0 / n, workspace=ws)  # epsilon/tau == 1: anti-CFL
    with pytest.raises(api.InvalidInput):
        dev.fast_f64(u, out, dd, 0.05, eta=-1e-3, workspace=ws)
    with pytest.raises(api.InvalidInput):
        dev.evolve(u, out, dd, 1.0 / (2 * n), 1, workspace=ws)  # epsilon/tau = 2
    with pytest.raises(api.InvalidInput):
        dev.build_kernel(n, 1.0 / n, 0.0)
    with pytest.raises(api.InvalidInput):
        dev.build_kernel(0, 0.05, 0.0)
    with pytest.raises(api.InvalidInput):
        dev.step_host(np.zeros((2, n)), np.zeros(2), 0.0)
    # a workspace too small for the batch is rejected, not overrun
    with pytest.raises(api.InvalidInput):
        dev.fast_f64(u, out, dd, 0.05, workspace=ws[:64])
    # nothing above left an error behind: a valid call still works
    dev.fast_f64(u, out, dd, 0.05, workspace=ws)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), np.zeros((2, n)))


def test_more_lines_than_one_grid_dimension(dev, orc, ref):
    """Batches of more than 65535 lines (a 256^3 tensor has 65536 lines per axis sweep): the line
    index is folded over two grid dimensions; every line of K2 (tiled and whole-line), the
    relaxed engine, the windowed K1 and the semi-discrete step equals the oracle's / the
    reference's, the last lines included."""
    import torch
    lines, n, tau = 65535 + 70, 8, 0.5
    rng = np.random.default_rng(65535)
    u = rng.uniform(-1, 1, (lines, n))
    drifts = rng.uniform(-1.5, 1.5, lines)
    k = [orc.kernel(n, tau, float(d)) for d in drifts[-80:]]
    # the last 80 lines (both sides of the fold) against the oracle, each with its own window
    K = np.ascontiguousarray(np.stack([x[0] for x in k]))
    first = np.array([x[1] for x in k], np.int64)
    want_tail = orc.direct(u[-80:], K, first, ktab_stride=2 * n + 1)
    du, dd = to_dev(u), to_dev(drifts)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    outs = {}
    for mode in (0, 2):  # tiled fast_kernel, whole-line K2L
        dev.set_fast_line(mode)
        o = torch.empty_like(du)
        bl = torch.empty(lines, dtype=torch.int64, device="cuda") if mode == 0 else None
        dev.fast_f64(du, o, dd, tau, blocks=bl, workspace=ws)
        torch.cuda.synchronize()
        outs[mode] = o.cpu().numpy()
        assert np.array_equal(outs[mode][-80:], want_tail), mode
    dev.set_fast_line(2)
    assert np.array_equal(outs[0], outs[2])
    # one shared window for the table engines
    kw, kfirst, _, _ = orc.kernel(n, tau, 0.25)
    kt = to_dev(kw)
    fr = torch.full((lines,), int(kfirst), dtype=torch.int64, device="cuda")
    want = orc.direct(u, kw, np.array([kfirst], np.int64))
    o = torch.empty_like(du)
    dev.relaxed_f64(du, o, kt, fr, 0.0)
    torch.cuda.synchronize()
    assert np.array_equal(o.cpu().numpy(), want)
    o2 = torch.empty_like(du)
    dev.fast_window_f64(du, o2, kt, fr[:1], tau, workspace=ws)
    torch.cuda.synchronize()
    assert np.array_equal(o2.cpu().numpy(), want)
    # windowed (wall) lines of m = 12 samples through the windowed K1: the last lines == the reference
    m = 12
    uw = rng.uniform(-1, 1, (lines, m))
    o3 = torch.empty((lines, m), dtype=torch.float64, device="cuda")
    dev.window_f64(to_dev(uw), o3, n, kt, fr[:1])
    torch.cuda.synchronize()
    got = o3.cpu().numpy()
    for l in (0, 65534, 65535, 65536, lines - 1):
        w, _, st = ref.kinetic_convolve(uw[l], n, tau, 0.25, periodic=False)
        assert st == 0 and np.array_equal(got[l], w), l
    # semi-discrete step with a zero potential == the fully discrete one (q = 1, V = 0)
    o4 = torch.empty_like(du)
    dev.step_semidiscrete(du, o4, kt, int(kfirst), 0.0, tau)
    torch.cuda.synchronize()
    assert np.array_equal(o4.cpu().numpy(), want)


@pytest.mark.parametrize("lines", [1, 3, 7, 9, 17])
@pytest.mark.parametrize("engine", [api.ENGINE_FAST, api.ENGINE_DIRECT, api.ENGINE_RELAXED])
def test_host_step_with_fewer_lines_than_pipeline_chunks(dev, orc, lines, engine):
    """lob_step_host_f64 pipelines the lines in 8 chunks: batches smaller than, equal to one more than,
    and not divisible by the chunk count give the oracle's step and block counts line by line."""
    n, tau = 512, 0.05
    rng = np.random.default_rng(lines)
    u = np.cumsum(rng.uniform(-2.0 / n, 2.0 / n, (lines, n)), axis=1)
    u -= np.linspace(0, 1, n, endpoint=False)[None, :] * u[:, -1:]
    drifts = rng.uniform(-1, 1, lines)
    v = np.cos(2 * np.pi * np.arange(n) / n)
    blocks = np.empty(lines, np.int64)
    got = dev.step_host(u, drifts, tau, tv=tau * v, engine=engine, blocks=blocks)
    ks = [orc.kernel(n, tau, float(d)) for d in drifts]
    K = np.ascontiguousarray(np.stack([k[0] for k in ks]))
    first = np.array([k[1] for k in ks], np.int64)
    want = orc.direct(u, K, first, tv=tau * v, ktab_stride=2 * n + 1)
    assert np.array_equal(got, want)
    assert list(blocks) == [orc.line_blocks(u[l]) for l in range(lines)]


@pytest.mark.parametrize("n,tau", [(64, 1.0 / (64 * 0.999)), (1000, 1.0 / (1000 * 0.97)), (64, 100.0), (512, 1e4),
                                   (4096, 1.0 / (4096 * 0.999))])
def test_time_steps_at_both_ends_of_the_anti_cfl_range(dev, ref, n, tau):
    """epsilon/tau just below the bound h0 = 1 (a window two samples wide in velocity) and a huge
    tau (a window so flat that its edges can hold minimisers: K2's gate sends those tiles to the
    direct formula): every engine == the reference's step."""
    lines = 3
    rng = np.random.default_rng(n)
    u = np.cumsum(rng.uniform(-1.0 / n, 1.0 / n, (lines, n)), axis=1) + 0.1 * np.sin(2 * np.pi * np.arange(n) / n)
    drifts = np.array([0.0, 0.37, -1.2])
    want, wb = ref.step_lines(u, tau, drifts, engine=1, nthreads=3)
    for name, got in all_engines(dev, u, drifts, tau).items():
        assert np.array_equal(got, want), name


@pytest.mark.parametrize("scale", [1e300, 1e150, 1e-290, 1e-310])
def test_extreme_magnitudes_through_every_engine(dev, ref, scale):
    """Lines scaled to the ends of the double range (overflowing fp32 screens and slope inversions,
    subnormal samples): every engine == the reference's step, infinities and all."""
    n, tau, lines = 1024, 0.05, 3
    rng = np.random.default_rng(7)
    u = (np.cumsum(rng.uniform(-1.0 / n, 1.0 / n, (lines, n)), axis=1) +
         np.sin(2 * np.pi * np.arange(n) / n)[None, :]) * scale
    drifts = np.array([0.5, -0.3, 1.1])
    want, _ = ref.step_lines(u, tau, drifts, engine=1, nthreads=3)
    for name, got in all_engines(dev, u, drifts, tau).items():
        assert np.array_equal(got, want), name


def test_contexts_on_concurrent_host_threads(dev):
    """One context per host thread (SURVEY 8b threading): four threads, each with its own context
    and stream, step different batches at once (K2 tiled with block counts, K2L, K1, the relaxed
    engine); every result == the same work done alone on the session's context."""
    import threading

    import torch
    n_long, n_short, tau, steps = 8192, 512, 0.02, 12

    def work(d, seed, stream):
        rng = np.random.default_rng(seed)
        res = {}
        for name, n in (("long", n_long), ("short", n_short)):
            lines = 6
            u = np.cumsum(rng.uniform(-1.0 / n, 1.0 / n, (lines, n)), axis=1) + np.sin(2 * np.pi * np.arange(n) / n)
            dr = rng.uniform(-1.5, 1.5, lines)
            with torch.cuda.stream(stream):
                a, b = to_dev(u), torch.empty((lines, n), dtype=torch.float64, device="cuda")
                dd = to_dev(dr)
                ws = torch.empty(d.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
                bl = torch.empty(lines, dtype=torch.int64, device="cuda")
                for i in range(steps):
                    d.fast_f64(a, b, dd, tau, blocks=bl, workspace=ws, flags=api.FAST_STATS_VALID if i else 0,
                               stream=stream)
                    a, b = b, a
                kt, fr = windows(d, n, tau, dr)
                o1, o2 = torch.empty_like(a), torch.empty_like(a)
                d.direct_f64(a, o1, kt, fr, ktab_stride=2 * n + 1, stream=stream)
                d.relaxed_f64(a, o2, kt, fr, 1e-6, ktab_stride=2 * n + 1, stream=stream)
                stream.synchronize()
                res[name] = (a.cpu().numpy(), bl.cpu().numpy(), o1.cpu().numpy(), o2.cpu().numpy())
        return res

    alone = [work(dev, 100 + t, torch.cuda.current_stream()) for t in range(4)]
    got, errs = [None] * 4, []

    def run(t):
        try:
            d = api.Device(0)
            try:
                got[t] = work(d, 100 + t, torch.cuda.Stream())
            finally:
                d.close()
        except Exception as exc:  # surfaced below
            errs.append(exc)

    threads = [threading.Thread(target=run, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errs, errs
    for t in range(4):
        for name in ("long", "short"):
            for x, y in zip(got[t][name], alone[t][name]):
                assert np.array_equal(x, y), (t, name)


@pytest.mark.parametrize("n", [256, 258, 260, 1000, 1002, 2044, 2046, 2048])
@pytest.mark.parametrize("offset", [0, 1])
def test_whole_line_kernel_bulk_and_register_loads(dev, orc, n, offset):
    """K2L loads a row by one TMA bulk copy when the row is even, 16-byte aligned and lands on an
    even shared-memory offset (n = 0 mod 4), else through registers: both paths, rows shifted by
    one sample off the 16-byte grid, lengths around the limits == the oracle."""
    import torch
    tau, lines = 0.02, 5
    rng = np.random.default_rng(n + offset)
    u = np.cumsum(rng.uniform(-1.0 / n, 1.0 / n, (lines, n)), axis=1) + 0.3 * np.sin(2 * np.pi * np.arange(n) / n)
    drifts = np.array([-1.1, -0.2, 0.0, 0.6, 1.7])
    buf = torch.zeros(lines * n + offset, dtype=torch.float64, device="cuda")
    du = buf[offset:].view(lines, n)
    du.copy_(to_dev(u))
    obuf = torch.zeros(lines * n + offset, dtype=torch.float64, device="cuda")
    out = obuf[offset:].view(lines, n)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    v = np.cos(2 * np.pi * np.arange(n) / n)
    dev.fast_f64(du, out, to_dev(drifts), tau, tv=to_dev(tau * v), workspace=ws)
    torch.cuda.synchronize()
    ks = [orc.kernel(n, tau, float(d)) for d in drifts]
    K = np.ascontiguousarray(np.stack([k[0] for k in ks]))
    first = np.array([k[1] for k in ks], np.int64)
    want = orc.direct(u, K, first, tv=tau * v, ktab_stride=2 * n + 1)
    assert np.array_equal(out.cpu().numpy(), want)
    c = dev.fast_counters(ws, lines, n)
    assert c["missed_outputs"] == 0, c


@pytest.mark.parametrize("seed", range(12))
def test_seeded_differential_sweep_of_engines(dev, orc, seed):
    """Seeded random shapes (length 1..3000, time step anywhere in the anti-CFL range, drifts up to
    |tau P| ~ 2.5, smooth / rough / piecewise-constant / kinked / spiky lines, a random potential):
    12 seeds x 8 cases, every engine (K1 screened and plain, K2 whole-line or tiled, the window-table
    K2, the relaxed engine at eta = 0) == the oracle's direct formula."""
    rng = np.random.default_rng(9000 + seed)
    for case in range(8):
        n = int(rng.choice([rng.integers(1, 40), rng.integers(40, 600), rng.integers(600, 3000)]))
        ratio = float(rng.uniform(0.02, 0.98))  # epsilon / tau
        tau = 1.0 / (n * ratio)
        lines = int(rng.integers(1, 6))
        x = np.arange(n) / n
        kind = int(rng.integers(0, 5))
        if kind == 0:
            u = np.sin(2 * np.pi * rng.integers(1, 5) * x)[None, :] * rng.uniform(0.1, 3.0, (lines, 1))
        elif kind == 1:
            u = np.cumsum(rng.uniform(-1, 1, (lines, n)), axis=1) / max(n, 1) ** 0.5
        elif kind == 2:
            u = np.floor(rng.uniform(0, 6, (lines, 1)) * x[None, :] * 4) * 0.25  # plateaus and jumps
        elif kind == 3:
            u = np.abs(x[None, :] - rng.uniform(0.2, 0.8, (lines, 1))) * rng.uniform(-3, 3, (lines, 1))  # kinks
        else:
            u = np.zeros((lines, n))
            u[np.arange(lines), rng.integers(0, n, lines)] = rng.uniform(-5, 5, lines)  # spikes
        u = np.ascontiguousarray(u + rng.uniform(-1e-9, 1e-9, (lines, n)) * (rng.random() < 0.5))
        drifts = rng.uniform(-2.5, 2.5, lines) / max(tau, 1e-300)
        drifts = np.clip(drifts, -50.0, 50.0)
        v = rng.uniform(-1, 1, n)
        ks = [orc.kernel(n, tau, float(d)) for d in drifts]
        K = np.ascontiguousarray(np.stack([k[0] for k in ks]))
        first = np.array([k[1] for k in ks], np.int64)
        want = orc.direct(u, K, first, tv=tau * v, ktab_stride=2 * n + 1)
        for name, got in all_engines(dev, u, drifts, tau, tv=tau * v).items():
            assert np.array_equal(got, want), (seed, case, name, n, tau, kind)


@pytest.mark.parametrize("n", [21, 64, 1024, 4096])
@pytest.mark.parametrize("tp", [2.5, 3.2, -4.5])
def test_window_centres_several_periods_away(dev, orc, n, tp):
    """|tau P| > 2: the window's centre lies more than two periods from the output, so the sources of
    the window-table K2 wrap three and more periods back (found by scripts/fuzz_engines.py: the
    wrap helper handled (-3n, 3n) only).  Smooth, spiky and rough lines, every engine == the oracle."""
    tau, lines = 4.0 / n, 3
    rng = np.random.default_rng(n)
    x = np.arange(n) / n
    u = np.stack([np.sin(2 * np.pi * x) * 0.7,
                  np.where(np.arange(n) == n // 3, 4.0, 0.0) + 1e-3 * x,
                  np.cumsum(rng.uniform(-1, 1, n)) / n ** 0.5])
    drifts = np.full(lines, tp / tau)
    v = rng.uniform(-1, 1, n)
    ks = [orc.kernel(n, tau, float(d)) for d in drifts]
    K = np.ascontiguousarray(np.stack([k[0] for k in ks]))
    first = np.array([k[1] for k in ks], np.int64)
    want = orc.direct(u, K, first, tv=tau * v, ktab_stride=2 * n + 1)
    for name, got in all_engines(dev, u, drifts, tau, tv=tau * v).items():
        assert np.array_equal(got, want), name


def test_seeded_differential_sweep_of_paths():
    """scripts/fuzz_paths.py, 24 seeds: evolve (resident and launch loop, both engines: states, block
    counts, drifts), the host step (every engine, eta 0 / 1e-7 / 1e-4) and the 2-D split step (direct
    and four fast layouts) on random sizes, time steps and drifts up to |tau P| = 4 == the reference."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "fuzz_paths.py"), "24"], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "failures: 0" in r.stdout and "checks: 288" in r.stdout, r.stdout[-2000:]


def test_seeded_sweep_of_random_convex_windows():
    """scripts/fuzz_windows.py, 30 seeds: the window-table K2 on random convex tables (sorted random
    slopes, a few distinct slopes with exact ties, quadratics centred in or outside the window, one
    kink; any first displacement) over random lines, three carried steps each == the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "fuzz_windows.py"), "30"], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "failures: 0" in r.stdout and "checks: 90" in r.stdout, r.stdout[-2000:]


def test_seeded_sweep_of_nd_split_and_tropical_gemm():
    """scripts/fuzz_nd.py, 20 seeds: split_step_nd on periodic tensors of rank 1-3 (every engine, the
    relaxed one with eta > 0, drifts up to |tau P| = 3) and on windowed tensors of ragged shapes
    (status and values), and the tropical GEMM with +inf entries == the reference."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "fuzz_nd.py"), "20"], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "failures: 0" in r.stdout and "checks: 120" in r.stdout, r.stdout[-2000:]


def test_seeded_sweep_of_long_lines_with_carried_statistics():
    """scripts/fuzz_long.py, 12 seeds: the tiled K2 on lines of 4096 .. 65536 samples (odd sizes too)
    mixing smooth modes, shocks, plateaus and noise, six consecutive steps on carried statistics
    (chained on alternate seeds), values and block counts == K1 at every step."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "fuzz_long.py"), "12"], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "failures: 0" in r.stdout and "checks: 72" in r.stdout, r.stdout[-2000:]
