"""K2 quick check on the GPU: K2 == K1 (bit-exact) on a set of line shapes with the
walk counters, then C2 / C5 step times.
usage: python scripts/k2_check.py [--lib LIB.so] [--no-check] [--c5]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--no-check", action="store_true")
ap.add_argument("--c5", action="store_true")
ap.add_argument("--pre", type=int, default=1000)
args = ap.parse_args()

import torch  # noqa: E402

from paper_1210_4090_b200 import _capi, api  # noqa: E402

if args.lib:
    _capi.LIB_PATH = os.path.abspath(args.lib)
dev = api.Device(0)


def k1(u, drifts, tau, tv):
    lines, n = u.shape
    ks = [dev.build_kernel(n, tau, float(p)) for p in drifts]
    kt = torch.from_numpy(np.stack([k.window for k in ks])).cuda()
    fi = torch.from_numpy(np.array([k.first for k in ks], np.int64)).cuda()
    out = torch.empty_like(u)
    dev.direct_f64(u, out, kt, fi, tv=tv, ktab_stride=2 * n + 1)
    return out


def k2(u, drifts, tau, tv, ws=None, flags=0):
    lines, n = u.shape
    if ws is None:
        ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(u)
    dev.fast_f64(u, out, torch.from_numpy(np.asarray(drifts, np.float64)).cuda(), tau, tv=tv, workspace=ws,
                 flags=flags)
    return out, ws


def check(name, u_np, drifts, tau, tv_np=None):
    u = torch.from_numpy(np.ascontiguousarray(u_np)).cuda()
    tv = None if tv_np is None else torch.from_numpy(tv_np).cuda()
    drifts = np.broadcast_to(np.asarray(drifts, np.float64), (u.shape[0],)).copy()
    a, ws = k2(u, drifts, tau, tv)
    b = k1(u, drifts, tau, tv)
    torch.cuda.synchronize()
    ok = torch.equal(a, b)
    c = dev.fast_counters(ws, u.shape[0], u.shape[1])
    bad = int((a != b).sum().item())
    print(json.dumps({"case": name, "equal": ok, "mismatch": bad, **c}), flush=True)
    return ok


if not args.no_check:
    rng = np.random.default_rng(1)
    allok = True
    for n, tau in [(24, 0.25), (600, 0.04), (1024, 0.05), (4096, 0.01)]:
        for drift in (0.0, 0.4, -0.7, 1.0):
            allok &= check(f"uniform n={n} P={drift}", rng.uniform(-1, 1, (4, n)), drift, tau)
    allok &= check("c3 lines", api.gen_c3_lines(0, 64, 4096), 0.0, 0.01)
    n = 4096
    x = np.arange(n) / n
    shapes = np.stack([np.zeros(n), np.where(x < 0.5, 0.0, 1.0), 1e8 * np.sin(2 * np.pi * x),
                       np.where(np.arange(n) == n // 3, -50.0, 0.0), np.where(np.arange(n) == n // 3, 50.0, 0.0),
                       1e-13 * rng.standard_normal(n), rng.uniform(-1, 1, n) * (x < 0.1)])
    for drift in (0.0, 0.85):
        allok &= check(f"structured P={drift}", shapes, drift, 0.01)
    # large drift: the window leaves the cached v_d table (|tau P| > 2)
    allok &= check("large drift", np.sin(2 * np.pi * np.arange(2048) / 2048)[None, :].repeat(2, 0), [150.0, -170.0],
                   0.02)
    # C2 after 60 steps, all 256 lines
    n, tau, L = 65536, 0.02, 256
    drifts = api.gen_c2_drifts(L)
    tvn = api.tau_v(api.gen_potential(2, n), tau)
    tv = torch.from_numpy(tvn).cuda()
    dd = torch.from_numpy(drifts).cuda()
    u = torch.zeros((L, n), dtype=torch.float64, device="cuda")
    v = torch.empty_like(u)
    ws = torch.empty(dev.fast_workspace_bytes(L, n), dtype=torch.uint8, device="cuda")
    for i in range(300):
        dev.fast_f64(u, v, dd, tau, tv=tv, workspace=ws, flags=api.FAST_STATS_VALID if i else 0)
        u, v = v, u
    torch.cuda.synchronize()
    print(json.dumps({"case": "c2 300 steps (chained counters)", **dev.fast_counters(ws, L, n)}), flush=True)
    allok &= check("c2 step 301", u.cpu().numpy(), drifts, tau, tvn)
    del u, v, ws
    # C5 20 steps on 4 lines
    n, tau = 1 << 20, 0.005
    u = torch.from_numpy(api.gen_c5_lines(0, 4, n)).cuda()
    v = torch.empty_like(u)
    tv5n = api.tau_v(api.gen_potential(3, n), tau)
    tv5 = torch.from_numpy(tv5n).cuda()
    d5 = torch.full((4,), 0.25, dtype=torch.float64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(4, n), dtype=torch.uint8, device="cuda")
    for i in range(20):
        dev.fast_f64(u, v, d5, tau, tv=tv5, workspace=ws, flags=api.FAST_STATS_VALID if i else 0)
        u, v = v, u
    torch.cuda.synchronize()
    allok &= check("c5 step 21", u.cpu().numpy(), [0.25] * 4, tau, tv5n)
    del u, v, ws
    print(json.dumps({"all_equal": bool(allok)}), flush=True)


def time_cfg(name, L, n, tau, drifts, tvn, u0, pre, reps=50):
    dd = torch.from_numpy(np.asarray(drifts, np.float64)).cuda()
    tv = torch.from_numpy(tvn).cuda()
    x = u0.clone()
    y = torch.empty_like(x)
    ws = torch.empty(dev.fast_workspace_bytes(L, n), dtype=torch.uint8, device="cuda")
    st = {"i": 0}

    def run(k):
        nonlocal x, y
        for _ in range(k):
            dev.fast_f64(x, y, dd, tau, tv=tv, workspace=ws,
                         flags=api.FAST_CHAINED | (api.FAST_STATS_VALID if st["i"] else 0))
            x, y = y, x
            st["i"] += 1

    run(pre)
    res = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        run(reps)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / reps)
    ms = min(res)
    out = {"case": name, "ms": sorted(res), "hbm_frac": L * n * 16 / (ms * 1e-3) / 6551e9}
    try:
        out.update(dev.fast_counters(ws, L, n))
    except Exception:
        pass
    print(json.dumps(out), flush=True)


n, tau, L = 65536, 0.02, 256
time_cfg("C2", L, n, tau, api.gen_c2_drifts(L), api.tau_v(api.gen_potential(2, n), tau),
         torch.zeros((L, n), dtype=torch.float64, device="cuda"), args.pre)
if args.c5:
    n, tau, L = 1 << 20, 0.005, 64
    time_cfg("C5", L, n, tau, np.full(L, 0.25), api.tau_v(api.gen_potential(3, n), tau),
             torch.from_numpy(api.gen_c5_lines(0, L, n)).cuda(), 20)
