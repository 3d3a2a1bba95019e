#!/usr/bin/env python
"""Full BASELINE.json configurations C1-C5 on one B200:
device-resident runs of every config at full size and step count, with
updates/s, roofline fractions and the parity checks each config admits at
full size:

  C1  2000 steps, K2 and K1 engines: final state / per-step blocks == the
      reference's evolve (tests/golden/c1_evolve.npz), H-bar.
  C2  5000 steps x 256 lines x N=65536 (K2): H-bar(P) per line; at sampled
      steps the K2 step == a K1 (direct, bit-exact) step of the same state,
      all 256 lines.  The same sweep at N=1024 is checked against the
      reference's H-bar (tests/golden/c2_hbar_n1024.npz).
  C3  K1 fp64 / fp32, 100 timed reps (median), lines 0-3 == reference golden.
  C4  500 split steps (x1 sweep, x2 sweep, potential) with the K1 and the K2
      sweep engines; the two trajectories must agree bit-for-bit; 20-step
      128^2 run == reference split_step_nd (tests/golden/c4_n128.npz).
  C5  200 steps x 64 lines x N=2^20 (K2); at sampled steps the K2 step == K1
      on 2 lines.

Writes one JSON document (default: profiles/r02_full_configs.json).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1210_4090_b200 import api  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


class Timer:
    def __init__(self, stream=None):
        self.s = torch.cuda.Event(enable_timing=True)
        self.e = torch.cuda.Event(enable_timing=True)
        self.stream = stream or torch.cuda.current_stream()

    def __enter__(self):
        torch.cuda.synchronize()
        self.s.record(self.stream)
        return self

    def __exit__(self, *a):
        self.e.record(self.stream)
        torch.cuda.synchronize()
        self.ms = self.s.elapsed_time(self.e)


def dev_t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def kernel_tables(dev, n, tau, drifts):
    ks = [dev.build_kernel(n, tau, float(p)) for p in drifts]
    return dev_t(np.stack([k.window for k in ks])), dev_t(np.array([k.first for k in ks], np.int64))


def direct_equals_fast(dev, u, drifts_h, tau, tv):
    """One K2 step vs one K1 step of the same device state (bit-exact)."""
    lines, n = u.shape
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    o_fast, o_dir = torch.empty_like(u), torch.empty_like(u)
    dev.fast_f64(u, o_fast, dev_t(drifts_h), tau, tv=tv, workspace=ws)
    kt, fi = kernel_tables(dev, n, tau, drifts_h)
    dev.direct_f64(u, o_dir, kt, fi, tv=tv, ktab_stride=2 * n + 1)
    torch.cuda.synchronize()
    return int((o_fast != o_dir).sum().item()), dev.fast_diagnostics(ws, lines, n)


def c1(dev):
    g = np.load(os.path.join(GOLD, "c1_evolve.npz"))
    n, tau, steps = 1024, 0.05, 2000
    out = {}
    for name, eng in (("k2_fast", api.ENGINE_FAST), ("k1_direct", api.ENGINE_DIRECT)):
        u = dev_t(g["u0"][None, :])
        scratch = torch.empty_like(u)
        sd = torch.empty(steps, dtype=torch.float64, device="cuda")
        sb = torch.empty(steps, dtype=torch.int64, device="cuda")
        ws = torch.empty(dev.fast_workspace_bytes(1, n), dtype=torch.uint8, device="cuda")
        tv = dev_t(api.tau_v(g["v"], tau))
        # one untimed step first: module loading and one-time kernel setup stay out of the timing
        w = dev_t(g["u0"][None, :])
        dev.evolve(w, torch.empty_like(w), dev_t(np.array([0.5])), tau, 1, tv=tv, engine=eng, workspace=ws)
        torch.cuda.synchronize()
        with Timer() as t:
            done = dev.evolve(u, scratch, dev_t(np.array([0.5])), tau, steps, tv=tv, engine=eng,
                              step_drift=sd, step_blocks=sb, workspace=ws)
        uf = u.cpu().numpy()[0]
        hbar = float(np.sum(uf - g["u0"]) / n / (steps * tau))
        out[name] = {"steps": done, "ms": t.ms, "updates_per_s": n * steps / (t.ms * 1e-3),
                     "final_state_bit_exact_vs_reference": bool(np.array_equal(uf, g["u_final"])),
                     "step_blocks_equal_reference": bool(np.array_equal(sb.cpu().numpy(), g["step_blocks"])),
                     "hbar": hbar, "hbar_reference": float(g["hbar"][0]),
                     "hbar_rel_err": abs(hbar - g["hbar"][0]) / abs(g["hbar"][0])}
    return out


def c2(dev, steps=5000, checks=(1, 1000, 2500, 4999)):
    n, lines, tau = 65536, 256, 0.02
    drifts_h = api.gen_c2_drifts(lines)
    drifts = dev_t(drifts_h)
    tv = dev_t(api.tau_v(api.gen_potential(2, n), tau))
    u0 = torch.zeros((lines, n), dtype=torch.float64, device="cuda")
    a, b = u0.clone(), torch.empty_like(u0)
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    blocks = torch.empty(lines, dtype=torch.int64, device="cuda")
    total_ms, chk = 0.0, []
    s = 0
    for stop in list(checks) + [steps]:
        if stop > s:
            with Timer() as t:
                for i in range(s, stop):
                    dev.fast_f64(a, b, drifts, tau, tv=tv, blocks=blocks, workspace=ws,
                                 flags=api.FAST_CHAINED | (api.FAST_STATS_VALID if i else 0))
                    a, b = b, a
            total_ms += t.ms
            s = stop
        if stop < steps:
            mism, miss = direct_equals_fast(dev, a, drifts_h, tau, tv)
            chk.append({"step": stop, "lines": lines, "k2_vs_k1_mismatches": mism, "k2_fallback_outputs": miss})
    uf = a.cpu().numpy()
    hbar = uf.sum(axis=1) / n / (steps * tau)
    bl = blocks.cpu().numpy()
    res = {"steps": steps, "ms": total_ms, "ms_per_step": total_ms / steps,
           "updates_per_s": lines * n * steps / (total_ms * 1e-3),
           "hbm_frac": lines * n * 16 * steps / (total_ms * 1e-3) / 1e9 / HBM,
           "finite": bool(np.isfinite(uf).all()), "k2_vs_k1_checks": chk,
           "hbar_P": {"P": drifts_h[::32].tolist(), "hbar": hbar[::32].tolist()},
           "hbar_min": float(hbar.min()), "hbar_max": float(hbar.max()),
           "blocks_per_line_final": {"mean": float(bl.mean()), "max": int(bl.max())}}
    # the same sweep at N=1024 against the reference's H-bar (5000 steps, all 256 lines)
    gp = os.path.join(GOLD, "c2_hbar_n1024.npz")
    if os.path.exists(gp):
        g = np.load(gp)
        nn = 1024
        u = torch.zeros((lines, nn), dtype=torch.float64, device="cuda")
        sc = torch.empty_like(u)
        wsn = torch.empty(dev.fast_workspace_bytes(lines, nn), dtype=torch.uint8, device="cuda")
        sb = torch.empty(steps, dtype=torch.int64, device="cuda")
        with Timer() as t:
            dev.evolve(u, sc, drifts, tau, steps, tv=dev_t(api.tau_v(g["v"], tau)), workspace=wsn)
        uf = u.cpu().numpy()
        hb = uf.sum(axis=1) / nn / (steps * tau)
        res["n1024_sweep_vs_reference"] = {
            "ms": t.ms, "hbar_max_rel_err": float(np.max(np.abs(hb - g["hbar"]) / np.abs(g["hbar"]))),
            "final_states_bit_exact": bool(np.array_equal(uf[g["keep"]], g["u_final"]))}
    return res


def c3(dev, reps=100):
    n, lines = 4096, 4096
    K = dev.build_kernel(n, 0.01, 0.0)
    u = dev_t(api.gen_c3_lines(0, lines, n))
    o = torch.empty_like(u)
    dk = dev_t(K.window)
    df = torch.full((lines,), K.first, dtype=torch.int64, device="cuda")
    cand = lines * n * (2 * n + 1)

    def med(fn):
        fn()
        ts = []
        for _ in range(reps):
            with Timer() as t:
                fn()
            ts.append(t.ms)
        return float(np.median(ts))

    fp = dev.bench_fp64()
    t64 = med(lambda: dev.direct_f64(u, o, dk, df))
    g = np.load(os.path.join(GOLD, "c3_lines0-3.npz"))
    exact = bool(np.array_equal(o[:4].cpu().numpy(), g["out"]))
    u32, o32 = u.float(), torch.empty_like(u, dtype=torch.float32)
    dk32 = dk.float()
    t32 = med(lambda: dev.direct_f32(u32, o32, dk32, df))
    return {"reps": reps, "fp64": {"ms_median": t64, "updates_per_s": lines * n / (t64 * 1e-3),
                                   "cand_per_s": cand / (t64 * 1e-3),
                                   "fp64_pipe_frac": 2 * cand / (t64 * 1e-3) / fp["dadd_ops_per_s"],
                                   "lines0_3_bit_exact_vs_reference": exact},
            "fp32": {"ms_median": t32, "updates_per_s": lines * n / (t32 * 1e-3), "cand_per_s": cand / (t32 * 1e-3)},
            "fp64_pipe_measured": fp}


def c4(dev, steps=500):
    n, tau = 2048, 0.01
    a = dev_t(api.gen_cos(n))
    res = {}
    finals = {}
    for name, eng, halves in (("k1_direct", api.ENGINE_DIRECT, 1), ("k2_fast", api.ENGINE_FAST, 2),
                              ("k2_fast_unfused", api.ENGINE_FAST, 1)):
        u = dev_t(api.gen_c4_u0(n))
        o, tmp = torch.empty_like(u), torch.empty_like(u)
        # two workspace halves: the fused four-launch step (transpose + statistics, sweep, x2)
        ws = torch.empty(halves * dev.fast_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
        bs = [api.c4_time_term(i * tau + tau) for i in range(steps)]
        # one untimed step on a scratch state: module loading and one-time engine setup stay out of the timing
        dev.split_step_2d(u.clone(), o, tmp, tau, 0.3, -0.7, a1=a, a2=a, b=bs[0], engine=eng, workspace=ws)
        with Timer() as t:
            for i in range(steps):
                dev.split_step_2d(u, o, tmp, tau, 0.3, -0.7, a1=a, a2=a, b=bs[i], engine=eng, workspace=ws)
                u, o = o, u
        finals[name] = u.cpu().numpy()
        res[name] = {"steps": steps, "ms": t.ms, "ms_per_step": t.ms / steps,
                     "updates_per_s": n * n * steps / (t.ms * 1e-3)}
        if eng == api.ENGINE_DIRECT:
            cand = 2 * n * n * (2 * n + 1) * steps
            res[name]["cand_per_s"] = cand / (t.ms * 1e-3)
    res["k1_k2_trajectories_bit_exact"] = bool(np.array_equal(finals["k1_direct"], finals["k2_fast"]) and
                                              np.array_equal(finals["k2_fast"], finals["k2_fast_unfused"]))
    res["mean_u_T_over_T"] = float(finals["k2_fast"].mean() / (steps * tau))
    gp = os.path.join(GOLD, "c4_n128.npz")
    if os.path.exists(gp):
        g = np.load(gp)
        m = 128
        am = dev_t(api.gen_cos(m))
        u = dev_t(g["u0"])
        o, tmp = torch.empty_like(u), torch.empty_like(u)
        ws = torch.empty(dev.fast_workspace_bytes(m, m), dtype=torch.uint8, device="cuda")
        ok = True
        k = 0
        for i in range(int(g["at"][-1]) + 1):
            dev.split_step_2d(u, o, tmp, tau, 0.3, -0.7, a1=am, a2=am, b=api.c4_time_term(i * tau + tau),
                              engine=api.ENGINE_FAST, workspace=ws)
            u, o = o, u
            if i == g["at"][k]:
                ok &= bool(np.array_equal(u.cpu().numpy(), g["states"][k]))
                k += 1
        res["n128_20steps_bit_exact_vs_reference"] = ok
    return res


def c5(dev, steps=200, checks=(1, 100, 199)):
    n, lines, tau, p = 1 << 20, 64, 0.005, 0.25
    t0 = time.perf_counter()
    a = dev_t(api.gen_c5_lines(0, lines, n))
    gen_s = time.perf_counter() - t0
    b = torch.empty_like(a)
    tv = dev_t(api.tau_v(api.gen_potential(3, n), tau))
    drifts = torch.full((lines,), p, dtype=torch.float64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    blocks = torch.empty(lines, dtype=torch.int64, device="cuda")
    total_ms, chk, s = 0.0, [], 0
    first_blocks = None
    for stop in list(checks) + [steps]:
        if stop > s:
            with Timer() as t:
                for i in range(s, stop):
                    dev.fast_f64(a, b, drifts, tau, tv=tv, blocks=blocks, workspace=ws,
                                 flags=api.FAST_CHAINED | (api.FAST_STATS_VALID if i else 0))
                    a, b = b, a
            total_ms += t.ms
            if first_blocks is None:
                first_blocks = blocks.cpu().numpy().copy()
            s = stop
        if stop < steps:
            sub = a[:2].contiguous()
            mism, miss = direct_equals_fast(dev, sub, np.full(2, p), tau, tv)
            chk.append({"step": stop, "lines": 2, "k2_vs_k1_mismatches": mism, "k2_fallback_outputs": miss})
    bl = blocks.cpu().numpy()
    # the same chained steps from the final state without StepStats (no block counts)
    x, y = a.clone(), torch.empty_like(a)
    nb = 20
    with Timer() as t:
        for i in range(nb):
            dev.fast_f64(x, y, drifts, tau, tv=tv, workspace=ws, flags=api.FAST_CHAINED | api.FAST_STATS_VALID)
            x, y = y, x
    del x, y
    return {"steps": steps, "ms": total_ms, "ms_per_step": total_ms / steps,
            "ms_per_step_without_block_counts": t.ms / nb,
            "updates_per_s": lines * n * steps / (total_ms * 1e-3),
            "hbm_frac": lines * n * 16 * steps / (total_ms * 1e-3) / 1e9 / HBM,
            "host_u0_generation_s": gen_s, "k2_vs_k1_checks": chk,
            "finite": bool(torch.isfinite(a).all().item()),
            "blocks_per_line_step0": {"mean": float(first_blocks.mean()), "max": int(first_blocks.max())},
            "blocks_per_line_final": {"mean": float(bl.mean()), "max": int(bl.max())}}


def c2_karp(dev, n=512, count=16):
    """C2's H-bar(P) two independent ways on the device at N = 512 (the period-matrix guard):
    the whole-period drift estimator (estimate_hbar_drift, K2 steps) and Karp's min-plus
    eigenvalue of the one-period matrix (build_period_matrix + eigenvalue_karp); the reference
    checks the same agreement at N = 128 (proj/tests/acceptance.cpp:351-366)."""
    tau = 0.02
    ell = int(round(1 / tau))
    v = api.gen_potential(2, n)
    tv = api.tau_v(v, tau)
    drifts = api.gen_c2_drifts(256)[np.linspace(0, 255, count).round().astype(int)]
    rows = []
    t0 = time.perf_counter()
    for P in drifts:
        est = dev.hbar_drift_host(np.zeros(n), float(P), tau, tv, api.ENGINE_FAST, 2000, 1e-11)
        k = dev.build_kernel(n, tau, float(P))
        kinc = dev_t(api.Device.period_kinetic(k))
        C = torch.empty((n, n), dtype=torch.float64, device="cuda")
        scr = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
        dev.period_matrix(kinc, dev_t(np.tile(tv, (ell, 1))), ell, C, scr)
        lam = dev.eigenvalue_karp(C)
        rows.append({"P": float(P), "drift_hbar": est["h_bar"], "karp_hbar": lam, "periods": est["n_steps"] // ell,
                     "converged": est["converged"], "abs_diff": abs(est["h_bar"] - lam)})
    return {"n": n, "tau": tau, "lines": rows, "max_abs_diff": max(r["abs_diff"] for r in rows),
            "seconds": time.perf_counter() - t0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_full_configs.json"))
    ap.add_argument("--only", default="c1,c2,c3,c4,c5,c2_karp")
    args = ap.parse_args()
    dev = api.Device(0)
    doc = {"device": torch.cuda.get_device_name(0), "hbm_peak_gbs": HBM}
    from bench import ClockSampler

    for name in args.only.split(","):
        t0 = time.perf_counter()
        clk = ClockSampler(0)
        clk.start()
        doc[name] = globals()[name](dev)
        doc[name]["clocks"] = clk.stop()
        doc[name]["wall_s"] = time.perf_counter() - t0
        print(name, json.dumps(doc[name])[:600], flush=True)
    with open(args.out, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
