#!/usr/bin/env python
"""Benchmark: Lax-Oleinik grid-point updates/s (fp64) on B200.

Workload (BASELINE.json configs[1], "C2"): 256 independent periodic lines of
N = 65536, per-line drift P_l = -2 + 4 l/255, tau = 0.02,
V = cos(2 pi x) + 0.5 cos(4 pi x + 1), u0 = 0.  One bench step = one fully
discrete Lax-Oleinik step of all 256 lines (step_fully_discrete: min-plus with
the kinetic kernel + potential; StepStats not requested, the API default, as C2's
H-bar needs none), run by the K2 fast exact engine, device-resident (u^{n+1}
feeds the next step).  The same step with decompose()'s block counts is timed
under config.with_block_counts_ms_per_step.
The state is first evolved `--presteps` steps (untimed) so the timed steps
see a developed, kinked solution like the bulk of C2's 5000 steps.
Working set 2 x 134 MB > 126 MB L2, so no L2 flush is needed.

--impl reference times the reference's own CPU implementation (oracle/_ref,
the laxol library built from its sources) on the box's host cores.

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Lax-Oleinik grid-point updates/s (fp64) at 1 GPU; % of FP64/HBM roofline"
N_SPACE, LINES, TAU = 65536, 256, 0.02
WORKLOAD = "C2: 256 lines x N=65536, P in [-2,2], tau=0.02, V=cos(2pi x)+0.5cos(4pi x+1), u0=0"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--presteps", type=int, default=1000)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="skip the per-kernel extra measurements")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--c4-dist", action="store_true",
                    help="N>1: also time the row-sharded C4 split step (P2P symmetric-memory exchange)")
    ap.add_argument("--ref-lines", type=int, default=0,
                    help="C2 lines per reference-arm step (default: one per host thread, <= 64)")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 7:
                for k, nm in enumerate(names):
                    if r[3 + k].lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        backend = "nccl" if args.impl == "b200" else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend, rank=rank, world_size=world)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_max(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- reference arm
def cpu_reference_rate(lines_sample: int, nthreads: int, engine: int = 1):
    """One step of `lines_sample` C2 lines through the reference library
    (oracle/_ref; step_fully_discrete per line on a std::thread pool).
    Returns (updates/s, seconds, sample description)."""
    from tests import _oracle

    ref = _oracle.reference()
    if ref is None:
        return None
    # inputs from the generators built into oracle/_ref: this arm maps no product library
    drifts = ref.gen_c2_drifts(LINES)
    idx = np.linspace(0, LINES - 1, lines_sample).round().astype(int)
    v = ref.gen_potential(2, N_SPACE)
    rng = np.random.default_rng(0)
    # the Naive engine's cost is data independent; a rough state stands in
    u = np.cumsum(rng.uniform(-1.0 / N_SPACE, 1.0 / N_SPACE, (lines_sample, N_SPACE)), axis=1)
    u -= np.linspace(0, 1, N_SPACE)[None, :] * u[:, -1:]
    t0 = time.perf_counter()
    ref.step_lines(u, TAU, drifts[idx], v=v, engine=engine, nthreads=nthreads, want_blocks=False)
    dt = time.perf_counter() - t0
    return lines_sample * N_SPACE / dt, dt, f"{lines_sample} C2 lines x 1 step, ConvEngine::Naive, {nthreads} threads"


REF_BUDGET_S = 150.0  # wall-clock budget of the reference arm (it must finish within minutes)


def config_for(world: int) -> dict:
    """The workload description both arms print (identical, so the driver can pair them)."""
    return {"workload": WORKLOAD, "lines": LINES, "n": N_SPACE, "tau": TAU,
            "l2": "working set 2 x 134 MB > 126 MB L2 (no flush needed)",
            "parallelism": f"C2's {LINES} lines partitioned over {world} GPU(s), {LINES // world} per GPU"
                           " (no per-step collective; H-bar(P) gathered at the end)"}


def run_reference(args, world, rank):
    """The reference's CPU path on all host threads.  One reference step of a C2 sample
    (one line per thread, ConvEngine::Naive) takes seconds, so the arm times at most
    as many steps as fit REF_BUDGET_S (after the requested warm-up steps) and reports
    the rate; `steps` is the number actually timed, `steps_requested` the driver's K."""
    if rank != 0:
        return
    nthreads = os.cpu_count() or 1
    lines_sample = args.ref_lines or max(1, min(nthreads, 64))
    rates, times = [], []
    t_start = time.perf_counter()
    warm = args.warmup
    i = 0
    while i < warm + args.steps:
        r = cpu_reference_rate(lines_sample, nthreads)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (reference build) missing"}))
            return
        if i >= warm:
            rates.append(r[0])
            times.append(r[1])
        i += 1
        elapsed = time.perf_counter() - t_start
        if rates and elapsed + r[1] > REF_BUDGET_S:
            break
    value = float(np.median(rates))
    line = {"metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": args.gpus, "steps": len(rates),
            "steps_requested": args.steps, "warmup": warm, "ms_per_step": float(np.median(times)) * 1e3,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_for(world),
            "impl_detail": {"engine": "reference laxol ConvEngine::Naive (CPU, oracle/_ref)",
                            "budget_s": REF_BUDGET_S, "sample": r[2]},
            "cpu_baseline": {"value": value, "unit": "updates/s", "cores": nthreads, "kind": "reference",
                             "sample": r[2]},
            "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ----------------------------------------------------------------------------- b200 arm
def run_b200(args, world, rank, local):
    import torch

    from paper_1210_4090_b200 import api

    torch.cuda.set_device(local)
    dev = api.Device(local)
    stream = torch.cuda.current_stream()
    # this rank's block of C2's lines (no per-step collective: the lines are independent)
    L = LINES // world
    l0 = rank * L
    dh = api.gen_c2_drifts(LINES)[l0:l0 + L].copy()
    drifts = torch.from_numpy(dh).cuda()
    tv_h = api.tau_v(api.gen_potential(2, N_SPACE), TAU)
    tv = torch.from_numpy(tv_h).cuda()
    a = torch.zeros((L, N_SPACE), dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    blocks = torch.empty(L, dtype=torch.int64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(L, N_SPACE), dtype=torch.uint8, device="cuda")
    st = {"cur": a, "nxt": b, "i": 0, "blocks": False}

    def step():
        # back-to-back device-resident steps: statistics carried over, per-line chaining
        dev.fast_f64(st["cur"], st["nxt"], drifts, TAU, tv=tv, blocks=blocks if st["blocks"] else None, workspace=ws,
                     flags=api.FAST_CHAINED | (api.FAST_STATS_VALID if st["i"] else 0), stream=stream)
        st["cur"], st["nxt"] = st["nxt"], st["cur"]
        st["i"] += 1

    for _ in range(args.presteps + args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = dev.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = dev.launches - launches0
    clk = clocks.stop()
    barrier(world)
    ms_max = allreduce_max(ms, world, device="cuda")
    updates = LINES * N_SPACE * args.steps  # the whole job: every rank's lines
    value = updates / (ms_max * 1e-3)
    hbm_peak, peak_kind = measured_peaks()
    per_launch_s = (ms / 1e3) / args.steps  # one fast_kernel launch per step
    achieved = L * N_SPACE * 16 / per_launch_s / 1e9
    finite = bool(torch.isfinite(st["cur"]).all().item())
    # H-bar(P) estimate per line, mean(u_T - u_0)/T (u_0 = 0), gathered on rank 0 over NCCL
    T = st["i"] * TAU
    hb = st["cur"].mean(dim=1) / T
    if world > 1:
        import torch.distributed as dist

        parts = [torch.empty_like(hb) for _ in range(world)]
        dist.all_gather(parts, hb)
        hb = torch.cat(parts)
    hb = hb.cpu().numpy()
    # the same step with decompose()'s block counts (StepStats requested), reported beside it
    st["blocks"] = True
    for _ in range(3):
        step()
    nb = 100
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(nb):
        step()
    e3.record(stream)
    torch.cuda.synchronize()
    ms_blocks = e2.elapsed_time(e3) / nb
    blocks_mean = float(blocks.double().mean().item())

    # ---- e2e: the host-buffer C-ABI entry (H2D + step + D2H every step) ----
    uh = torch.empty((L, N_SPACE), dtype=torch.float64, pin_memory=True)
    uh.copy_(st["cur"])
    oh = torch.empty_like(uh, pin_memory=True)
    un, on = uh.numpy(), oh.numpy()
    e2e_steps = max(1, min(args.steps, 10))
    dev.step_host(un, dh, TAU, tv=tv_h, out=on)  # warm
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        dev.step_host(un, dh, TAU, tv=tv_h, out=on)
        un, on = on, un
    dt = allreduce_max(time.perf_counter() - t0, world, device="cuda")
    e2e = {"value": LINES * N_SPACE * e2e_steps / dt, "unit": "updates/s",
           "h2d_bytes_per_step": int(L * N_SPACE * 8 + L * 8 + N_SPACE * 8),
           "d2h_bytes_per_step": int(L * N_SPACE * 8),
           "steps": e2e_steps, "api": "lob_step_host_f64 (pinned host buffers), per GPU"}
    # the e2e roofline: the same bytes moved by plain copies alone (H2D and D2H on two
    # streams at once, pinned buffers, no compute) - the host link bounds the e2e number
    dbuf_in = torch.empty_like(uh, device="cuda")
    dbuf_out = torch.empty_like(uh, device="cuda")
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    for rep in range(e2e_steps + 1):
        if rep == 1:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
        with torch.cuda.stream(s_in):
            dbuf_in.copy_(uh, non_blocking=True)
        with torch.cuda.stream(s_out):
            oh.copy_(dbuf_out, non_blocking=True)
    torch.cuda.synchronize()
    dtc = allreduce_max(time.perf_counter() - t0, world, device="cuda")
    bound = LINES * N_SPACE * e2e_steps / dtc
    e2e["copy_bound"] = {"value": bound, "unit": "updates/s", "frac": e2e["value"] / bound,
                         "what": "concurrent pinned H2D + D2H of one step's state, no compute"}
    del dbuf_in, dbuf_out, a, b, ws
    # e2e through the C++ API a reference user calls (Engine::step_fully_discrete, one pageable
    # std::vector line per call, V evaluated per point on the host like the reference)
    exe = os.path.join(ROOT, "tests", "cpp", "test_engine")
    if world == 1 and os.path.exists(exe):
        try:
            r = subprocess.run([exe, "--bench", "16"], capture_output=True, text=True, timeout=300)
            e2e["cpp_api_pageable"] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as exc:  # reported, not fatal
            e2e["cpp_api_pageable"] = {"error": str(exc)[:200]}
    st.clear()
    torch.cuda.empty_cache()
    # the row-sharded C4 split step across the ranks (every rank takes part)
    c4d = c4_dist_workload(dev, world, rank) if world > 1 and args.c4_dist else None

    if rank != 0:
        return
    traffic = None
    tp = os.path.join(ROOT, "profiles", "k2_c2_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("bytes_per_launch")
    line = {
        "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C2 generators, include/laxol_b200_configs.h)",
        "config": config_for(world),
        "impl_detail": {"engine": "K2 fast exact min-plus (LOB_ENGINE_FAST), chained steps",
                        "presteps": args.presteps, "lines_per_gpu": L, "state_finite": finite,
                        "step_stats": "not requested (step_fully_discrete's default)",
                        "with_block_counts_ms_per_step": ms_blocks, "mean_blocks_per_line": blocks_mean,
                        "hbar_gathered": {"lines": int(hb.size), "T": T, "min": float(hb.min()),
                                          "max": float(hb.max()), "finite": bool(np.isfinite(hb).all())}},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                     "algorithmic_bytes_per_update": 16},
        "clocks": clk, "gpu_launches": int(launches), "e2e": e2e,
    }
    if not args.no_cpu_baseline and world == 1:
        nthreads = os.cpu_count() or 1
        r = cpu_reference_rate(max(1, min(nthreads, 64)), nthreads)
        if r is not None:
            line["cpu_baseline"] = {"value": r[0], "unit": "updates/s", "cores": nthreads, "kind": "reference",
                                    "sample": r[2], "seconds": r[1]}
    if world == 1:
        line["c5"] = c5_workload(dev, hbm_peak)
        line["c4"] = c4_workload(dev, hbm_peak)
    if c4d is not None:
        line["c4_dist"] = c4d
    if not args.no_extras and world == 1:
        line["kernels"] = extras(dev)
    print(json.dumps(line))


def c5_workload(dev, hbm_peak):
    """C5 (configs[4], the largest per-step config): 64 lines x N=2^20, tau=0.005, P=0.25,
    V=0.5 sin(2 pi x), u0 = 64 random Fourier modes; K2 steps after 20 untimed ones."""
    import torch

    from paper_1210_4090_b200 import api

    n, tau, L = 1 << 20, 0.005, 64
    cur = torch.from_numpy(api.gen_c5_lines(0, L, n)).cuda()
    nxt = torch.empty_like(cur)
    tv = torch.from_numpy(api.tau_v(api.gen_potential(3, n), tau)).cuda()
    dd = torch.full((L,), 0.25, dtype=torch.float64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(L, n), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    k = 0

    def run(m):
        nonlocal cur, nxt, k
        for _ in range(m):
            dev.fast_f64(cur, nxt, dd, tau, tv=tv, workspace=ws,
                         flags=api.FAST_CHAINED | (api.FAST_STATS_VALID if k else 0), stream=stream)
            cur, nxt = nxt, cur
            k += 1

    run(20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 50
    e0.record(stream)
    run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    c = dev.fast_counters(ws, L, n)
    ach = L * n * 16 / (ms * 1e-3) / 1e9
    out = {"workload": "C5: 64 lines x N=2^20, tau=0.005, P=0.25, V=0.5 sin(2 pi x), 64 random modes",
           "ms_per_step": ms, "updates_per_s": L * n / (ms * 1e-3), "steps": steps, "presteps": 20,
           "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak},
           "walk_tiles": c["tiles"] - c["direct_tiles_gate"] - c["direct_tiles_heavy"], "tiles": c["tiles"]}
    del cur, nxt, ws
    torch.cuda.empty_cache()
    return out


def c4_workload(dev, hbm_peak):
    """C4 (configs[3]): 2-D periodic torus 2048^2 by dimension splitting, P=(0.3,-0.7),
    V=cos(2 pi x1)cos(2 pi x2)+0.2 sin(2 pi t) at the arrival time, u0=sin(2 pi x1)+cos(2 pi x2),
    tau=0.01; split steps (x1 sweep, x2 sweep, tau*V) through lob_split_step_2d_f64 with the
    fast engine after 20 untimed steps.  One update = one tensor point per split step; the
    roofline counts 16 algorithmic bytes per point (read u, write u^{n+1}); the 32 MB state
    is L2-resident, so the fraction is of HBM bandwidth, not the binding limit."""
    import torch

    from paper_1210_4090_b200 import api

    n, tau = 2048, 0.01
    am = torch.from_numpy(api.gen_cos(n)).cuda()
    u = torch.from_numpy(api.gen_c4_u0(n)).cuda()
    o, t = torch.empty_like(u), torch.empty_like(u)
    ws = torch.empty(2 * dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    k = 0

    def run(m):
        nonlocal u, o, k
        for _ in range(m):
            dev.split_step_2d(u, o, t, tau, 0.3, -0.7, a1=am, a2=am, b=api.c4_time_term(k * tau + tau),
                              engine=api.ENGINE_FAST, workspace=ws, stream=stream)
            u, o = o, u
            k += 1

    run(20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 100
    e0.record(stream)
    run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ach = n * n * 16 / (ms * 1e-3) / 1e9
    out = {"workload": "C4: 2048^2 torus, dimension splitting, P=(0.3,-0.7), V=cos cos + 0.2 sin 2 pi t, tau=0.01",
           "ms_per_step": ms, "updates_per_s": n * n / (ms * 1e-3), "steps": steps, "presteps": 20,
           "path": "transpose -> K2L row sweep -> transpose -> K2L row sweep with tau*V in its epilogue",
           "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                        "note": "32 MB state resident in the 126 MB L2"}}
    del u, o, t, ws
    torch.cuda.empty_cache()
    return out


def c4_dist_workload(dev, world, rank):
    """C4 (2048^2, P=(0.3,-0.7), V=cos cos + 0.2 sin 2 pi t, tau=0.01) sharded by rows over the
    ranks (paper_1210_4090_b200/dist.py): per step two row-slab exchanges around K2L sweeps.  The
    exchange runs over NVLink peer memory (CUDA symmetric memory, one push-transpose kernel per
    exchange) when every rank can set it up, else NCCL all-to-all between pack / unpack kernels.
    Timed with CUDA events, max over ranks; 16 updates-bytes per point and step as for c4."""
    import torch
    import torch.distributed as dist

    from paper_1210_4090_b200 import api
    from paper_1210_4090_b200.dist import P2PExchange, split_step_2d_dist

    n, tau, steps = 2048, 0.01, 50
    b = n // world
    out = {"workload": "C4 2048^2 row-sharded over the ranks", "rows_per_rank": b}
    try:
        p2p, err = None, ""
        try:
            p2p = P2PExchange(dev, b, n)
        except Exception as exc:  # decided collectively below
            err = str(exc)[:160]
        ok = torch.tensor([1 if p2p is not None else 0], dtype=torch.int32, device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not int(ok.item()):
            p2p = None
        out["exchange"] = "p2p symmetric-memory push (lob_slab_push_f64)" if p2p else \
            ("nccl all_to_all" + (f" (p2p unavailable: {err})" if err else " (p2p unavailable on a peer)"))
        u0 = api.gen_c4_u0(n)
        a = api.gen_cos(n)
        v = torch.from_numpy(np.ascontiguousarray(u0[rank * b:(rank + 1) * b])).cuda()
        wss = {}
        k = 0

        def run(m):
            nonlocal v, k
            for _ in range(m):
                v = split_step_2d_dist(dev, v, tau, 0.3, -0.7, a1=a, a2=a, b=api.c4_time_term((k + 1) * tau),
                                       engine=api.ENGINE_FAST, workspaces=wss, p2p=p2p)
                k += 1

        run(5)
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(steps)
        e1.record()
        torch.cuda.synchronize()
        ms = allreduce_max(e0.elapsed_time(e1) / steps, world, device="cuda")
        out.update({"ms_per_step": ms, "updates_per_s": n * n / (ms * 1e-3), "steps": steps,
                    "finite": bool(torch.isfinite(v).all().item())})
    except Exception as exc:  # reported, not fatal
        out["error"] = str(exc)[:200]
    return out


def extras(dev):
    """Secondary measurements: K1 direct (C3) against the FP64 pipe, K2 on C3/C5."""
    import torch

    from paper_1210_4090_b200 import api

    out = {}
    fp = dev.bench_fp64()
    out["fp64_pipe_measured"] = fp
    ev = lambda: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))  # noqa: E731

    def timeit(fn, reps):
        fn()
        torch.cuda.synchronize()
        s, e = ev()
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps * 1e-3

    n = 4096
    K = dev.build_kernel(n, 0.01, 0.0)
    u = torch.from_numpy(api.gen_c3_lines(0, 4096, n)).cuda()
    o = torch.empty_like(u)
    dk = torch.from_numpy(K.window).cuda()
    df = torch.full((4096,), K.first, dtype=torch.int64, device="cuda")
    cand = 4096 * 4096 * (2 * n + 1)
    dev.set_direct_mode(api.DIRECT_PLAIN)
    t = timeit(lambda: dev.direct_f64(u, o, dk, df), 5)
    out["k1_direct_c3_f64_plain"] = {
        "ms": t * 1e3, "updates_per_s": 4096 * 4096 / t, "cand_per_s": cand / t,
        "roofline": {"bound": "fp64 pipe", "ops_per_candidate": 2, "achieved_ops": 2 * cand / t,
                     "peak_ops": fp["dadd_ops_per_s"], "frac": 2 * cand / t / fp["dadd_ops_per_s"],
                     "frac_of_minplus_mix_peak": cand / t / fp["minplus_cand_per_s"]}}
    dev.set_direct_mode(api.DIRECT_SCREENED)
    dev.direct_fallbacks(reset=True)
    t = timeit(lambda: dev.direct_f64(u, o, dk, df), 5)
    # the screened sweep runs on the FP32 pipes: one FADD (FMA pipe, 128 lanes/SM/clk) and half
    # an FMNMX3 (ALU pipe, 64 lanes/SM/clk) per candidate -> both ceilings are 128 cand/SM/clk
    import torch as _t
    fp32_peak = _t.cuda.get_device_properties(0).multi_processor_count * 128 * fp["sm_clock_ghz"] * 1e9
    out["k1_direct_c3_f64"] = {
        "ms": t * 1e3, "updates_per_s": 4096 * 4096 / t, "cand_per_s": cand / t,
        "impl": "fp32 screen + fp64 re-evaluation (bit-identical; LOB_DIRECT_SCREENED, the default)",
        "full_fp64_outputs_per_call": dev.direct_fallbacks() / 6,
        "roofline": {"bound": "fp32 issue (FADD on the FMA pipe + FMNMX3 on the ALU pipe per 2 candidates)",
                     "achieved_cand_per_s": cand / t, "peak_cand_per_s": fp32_peak, "frac": cand / t / fp32_peak}}
    u32, o32, dk32 = u.float(), torch.empty_like(u.float()), dk.float()
    t = timeit(lambda: dev.direct_f32(u32, o32, dk32, df), 5)
    out["k1_direct_c3_f32"] = {"ms": t * 1e3, "updates_per_s": 4096 * 4096 / t, "cand_per_s": cand / t,
                               "roofline": {"bound": "fp32 issue", "peak_cand_per_s": fp32_peak,
                                            "frac": cand / t / fp32_peak}}
    ws = torch.empty(dev.fast_workspace_bytes(4096, n), dtype=torch.uint8, device="cuda")
    z = torch.zeros(4096, dtype=torch.float64, device="cuda")
    t = timeit(lambda: dev.fast_f64(u, o, z, 0.01, workspace=ws), 10)
    out["k2_fast_c3"] = {"ms": t * 1e3, "updates_per_s": 4096 * 4096 / t,
                         "hbm_frac": 4096 * 4096 * 16 / t / 1e9 / measured_peaks()[0]}
    del u, o, u32, o32, ws

    # C2 through the reference's evolve API (lob_evolve_f64: per-step drift and block counts fused)
    st = torch.zeros((LINES, N_SPACE), dtype=torch.float64, device="cuda")
    scr = torch.empty_like(st)
    dr = torch.from_numpy(api.gen_c2_drifts(LINES)).cuda()
    tvd = torch.from_numpy(api.tau_v(api.gen_potential(2, N_SPACE), TAU)).cuda()
    wse = torch.empty(dev.fast_workspace_bytes(LINES, N_SPACE), dtype=torch.uint8, device="cuda")
    dev.evolve(st, scr, dr, TAU, 200, tv=tvd, workspace=wse)
    ne = 500  # one evolve call of 500 steps (C2 runs as one call of 5000)
    sd = torch.empty(ne * LINES, dtype=torch.float64, device="cuda")
    sb = torch.empty(ne * LINES, dtype=torch.int64, device="cuda")
    t = timeit(lambda: dev.evolve(st, scr, dr, TAU, ne, tv=tvd, step_drift=sd, step_blocks=sb, workspace=wse), 1)
    out["c2_evolve_api"] = {"ms_per_step": t * 1e3 / ne, "updates_per_s": LINES * N_SPACE * ne / t,
                            "includes": "per-step drift and decompose block counts (proj/src/scheme.cpp:208-272)"}
    del st, scr, wse

    # weak-KAM consumers: tropical product at the dense guard n = 512, Karp, period matrix
    m = 512
    rng = np.random.default_rng(0)
    A = torch.from_numpy(rng.uniform(-1, 1, (m, m))).cuda()
    B = torch.from_numpy(rng.uniform(-1, 1, (m, m))).cuda()
    C = torch.empty_like(A)
    t = timeit(lambda: dev.minplus_gemm(A, B, C), 20)
    out["minplus_product_512"] = {"ms": t * 1e3, "cand_per_s": m ** 3 / t,
                                  "frac_of_minplus_mix_peak": m ** 3 / t / fp["minplus_cand_per_s"]}
    dev.eigenvalue_karp(A)
    t0 = time.perf_counter()
    dev.eigenvalue_karp(A)
    out["eigenvalue_karp_512"] = {"ms": (time.perf_counter() - t0) * 1e3,
                                  "impl": "one 16-CTA cluster launch (C in shared memory, D rows via DSMEM)"}
    kinc = torch.from_numpy(api.Device.period_kinetic(dev.build_kernel(m, 0.125, 0.3))).cuda()
    tvs = torch.from_numpy(np.tile(0.125 * api.gen_potential(1, m), (8, 1))).cuda()
    scratch = torch.empty(2 * m * m, dtype=torch.float64, device="cuda")
    t = timeit(lambda: dev.period_matrix(kinc, tvs, 8, C, scratch), 5)
    out["period_matrix_512_ell8"] = {"ms": t * 1e3, "cand_per_s": 7 * m ** 3 / t}
    # step_semidiscrete: C1's grid and V = cos(2 pi x) = potential_cosine(0, -1, 1), q = 4
    n1, tau1 = 1024, 0.05
    k1 = dev.build_kernel(n1, tau1, 0.5)
    us = torch.from_numpy(api.gen_sin(n1)[None, :].repeat(64, 0)).cuda()
    os_ = torch.empty_like(us)
    kt = torch.from_numpy(k1.window).cuda()
    pot = api.potential_cosine(0.0, -1.0, 1)
    t = timeit(lambda: dev.step_semidiscrete(us, os_, kt, k1.first, 0.0, tau1, pot, 4), 3)
    out["semidiscrete_c1x64_q4"] = {"ms": t * 1e3, "lines": 64, "n": n1,
                                    "cand_per_s": 64 * n1 * (2 * n1 + 1) / t}
    return out


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_b200(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
