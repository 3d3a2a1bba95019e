"""Seeded sweep of the window-table K2 (lob_minplus_fast_window_f64: any convex window) with
random convex tables - sorted random slopes, flat runs (ties), piecewise-linear and
quadratic-like shapes, minima anywhere incl. at an edge, any first displacement - on random
lines, one step and carried steps (LOB_FAST_STATS_VALID), against the oracle's direct formula.
usage: fuzz_windows.py [seeds]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from tests import _oracle
from paper_1210_4090_b200 import api

dev = api.Device(0)
orc = _oracle.oracle()
nseeds = int(sys.argv[1]) if len(sys.argv) > 1 else 100
fails = checks = 0


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


for seed in range(nseeds):
    rng = np.random.default_rng(40000 + seed)
    n = int(rng.choice([rng.integers(2, 40), rng.integers(40, 700), rng.integers(700, 5000)]))
    lines = int(rng.integers(1, 5))
    W = 2 * n + 1
    shape = int(rng.integers(0, 4))
    K = np.empty((lines, W))
    first = np.empty(lines, np.int64)
    for l in range(lines):
        if shape == 0:    # sorted random slopes
            s = np.sort(rng.normal(0, rng.uniform(1e-4, 1.0), W - 1))
        elif shape == 1:  # few distinct slopes: long flat-slope runs, exact ties
            s = np.sort(rng.choice(rng.integers(-4, 5, 6) * 2.0 ** -int(rng.integers(0, 12)), W - 1))
        elif shape == 2:  # quadratic-like with a random centre (possibly outside the window)
            c = rng.uniform(-0.3, 1.3) * W
            s = (np.arange(W - 1) + 0.5 - c) * rng.uniform(1e-6, 1e-2)
        else:             # absolute value: one kink
            c = int(rng.integers(0, W))
            s = np.where(np.arange(W - 1) < c, -1.0, 1.0) * rng.uniform(1e-3, 1.0)
        K[l] = np.concatenate([[0.0], np.cumsum(s)]) + rng.uniform(-1, 1)
        first[l] = int(rng.integers(-3 * n, 2 * n))
    x = np.arange(n) / n
    kind = int(rng.integers(0, 4))
    if kind == 0:
        u = np.sin(2 * np.pi * rng.integers(1, 4) * x)[None, :] * rng.uniform(0.01, 2.0, (lines, 1))
    elif kind == 1:
        u = np.cumsum(rng.uniform(-1, 1, (lines, n)), axis=1) * rng.uniform(1e-4, 0.1)
    elif kind == 2:
        u = np.round(rng.uniform(-2, 2, (lines, n)) * 4) / 4  # heavy ties
    else:
        u = np.zeros((lines, n)) + rng.uniform(-1, 1, (lines, 1))
    u = np.ascontiguousarray(u)
    tv = rng.uniform(-0.1, 0.1, n)
    tau = 1.0 / (n * 0.5)
    du, o = t(u), torch.empty((lines, n), dtype=torch.float64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    dk, df, dtv = t(K), t(first), t(tv)
    cur = u
    for step in range(3):  # carried statistics on steps 1 and 2
        want = orc.direct(cur, K, first, tv=tv, ktab_stride=W)
        try:
            dev.fast_window_f64(du, o, dk, df, tau, tv=dtv, workspace=ws, ktab_stride=W,
                                flags=api.FAST_STATS_VALID if step else 0)
            torch.cuda.synchronize()
        except Exception as exc:
            fails += 1
            print("EXC", seed, step, n, shape, kind, str(exc)[:200], flush=True)
            break
        checks += 1
        got = o.cpu().numpy()
        if not np.array_equal(got, want):
            fails += 1
            bad = np.argwhere(got != want)
            print("FAIL", seed, "step", step, "n", n, "shape", shape, "kind", kind, "first", first.tolist(),
                  "bad", len(bad), bad[:3].tolist(), dev.fast_counters(ws, lines, n), flush=True)
            break
        cur = want
        du, o = o, du
print("done, checks:", checks, "failures:", fails)
