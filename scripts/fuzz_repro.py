"""Reproduce one case of tests/test_edge_cases_gpu.py::test_seeded_differential_sweep_of_engines
(seed, case) and print where the window-table K2 differs from the oracle, with its counters."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from tests import _oracle
from paper_1210_4090_b200 import api

seed, want_case = int(sys.argv[1]), int(sys.argv[2])
dev = api.Device(0)
orc = _oracle.oracle()
rng = np.random.default_rng(9000 + seed)
for case in range(8):
    n = int(rng.choice([rng.integers(1, 40), rng.integers(40, 600), rng.integers(600, 3000)]))
    ratio = float(rng.uniform(0.02, 0.98))
    tau = 1.0 / (n * ratio)
    lines = int(rng.integers(1, 6))
    x = np.arange(n) / n
    kind = int(rng.integers(0, 5))
    if kind == 0:
        u = np.sin(2 * np.pi * rng.integers(1, 5) * x)[None, :] * rng.uniform(0.1, 3.0, (lines, 1))
    elif kind == 1:
        u = np.cumsum(rng.uniform(-1, 1, (lines, n)), axis=1) / max(n, 1) ** 0.5
    elif kind == 2:
        u = np.floor(rng.uniform(0, 6, (lines, 1)) * x[None, :] * 4) * 0.25
    elif kind == 3:
        u = np.abs(x[None, :] - rng.uniform(0.2, 0.8, (lines, 1))) * rng.uniform(-3, 3, (lines, 1))
    else:
        u = np.zeros((lines, n))
        u[np.arange(lines), rng.integers(0, n, lines)] = rng.uniform(-5, 5, lines)
    u = np.ascontiguousarray(u + rng.uniform(-1e-9, 1e-9, (lines, n)) * (rng.random() < 0.5))
    drifts = np.clip(rng.uniform(-2.5, 2.5, lines) / max(tau, 1e-300), -50.0, 50.0)
    v = rng.uniform(-1, 1, n)
    if case != want_case:
        continue
    ks = [orc.kernel(n, tau, float(d)) for d in drifts]
    K = np.ascontiguousarray(np.stack([k[0] for k in ks]))
    first = np.array([k[1] for k in ks], np.int64)
    want = orc.direct(u, K, first, ktab_stride=2 * n + 1)
    du = torch.from_numpy(u).cuda()
    for mode in (2, 0):
        dev.set_fast_line(mode)
        ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
        o = torch.empty_like(du)
        dev.fast_window_f64(du, o, torch.from_numpy(K).cuda(), torch.from_numpy(first).cuda(), tau, workspace=ws,
                            ktab_stride=2 * n + 1)
        torch.cuda.synchronize()
        got = o.cpu().numpy()
        bad = np.argwhere(got != want)
        print("mode", mode, "n", n, "tau", tau, "lines", lines, "kind", kind, "drifts", drifts, "first", first)
        print("counters", dev.fast_counters(ws, lines, n))
        for l, j in bad[:10]:
            w = K[l]
            cands = np.array([u[l, (j - first[l] - k) % n] + w[k] for k in range(2 * n + 1)])
            print(" line", l, "j", j, "got", got[l, j], "want", want[l, j], "argmin w", int(np.argmin(cands)),
                  "d", int(first[l] + np.argmin(cands)))
    dev.set_fast_line(2)
    # which (source, window index) pair gives each wrong value, and where it belongs
    for l, j in bad[:4]:
        w = K[l]
        hits = [(y, k) for y in range(n) for k in range(2 * n + 1) if u[l, y] + w[k] == got[l, j]]
        print(" wrong value at line", l, "j", j, "equals u[y] + K[k] for (y, k, d, (y+d)%n):",
              [(y, k, int(first[l] + k), int((y + first[l] + k) % n)) for y, k in hits][:6])
