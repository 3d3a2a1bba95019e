"""Seeded sweep of the tiled K2 on long lines with carried statistics: random mixes of smooth
modes, kinks (shocks), plateaus and rough noise, n in {4096 .. 65536 (+ odd sizes)}, random time
step and drifts (|tau P| up to 2.6), 6 consecutive steps with LOB_FAST_STATS_VALID (chained on
alternate seeds), block counts on; every step == K1 (itself pinned to the oracle) with the walk
counters reported.  usage: fuzz_long.py [seeds]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1210_4090_b200 import api

dev = api.Device(0)
nseeds = int(sys.argv[1]) if len(sys.argv) > 1 else 24
fails = checks = 0
for seed in range(nseeds):
    rng = np.random.default_rng(80000 + seed)
    n = int(rng.choice([4096, 5000, 8191, 16384, 40000, 65536]))
    lines = int(rng.integers(1, 5))
    tau = 1.0 / (n * float(rng.uniform(0.01, 0.9)))
    tp = rng.uniform(-2.6, 2.6, lines) if rng.random() < 0.4 else rng.uniform(-1.5, 1.5, lines)
    drifts = tp / tau
    x = np.arange(n) / n
    u = np.zeros((lines, n))
    for l in range(lines):
        for _ in range(int(rng.integers(1, 4))):
            k = int(rng.integers(0, 4))
            if k == 0:
                u[l] += np.sin(2 * np.pi * rng.integers(1, 40) * x + rng.uniform(0, 6)) * rng.uniform(0.01, 1.0)
            elif k == 1:
                u[l] += -np.abs(x - rng.uniform(0.1, 0.9)) * rng.uniform(0.1, 4.0)  # a concave kink (shock)
            elif k == 2:
                u[l] += np.floor(x * rng.integers(2, 30)) * rng.uniform(-0.05, 0.05)  # plateaus, jumps
            else:
                u[l] += np.cumsum(rng.uniform(-1, 1, n)) * rng.uniform(1e-7, 1e-3)
    u *= tau * float(rng.uniform(0.2, 3.0)) * 10  # scale slopes against the window's
    v = np.cos(2 * np.pi * x) * rng.uniform(0, 1.0) + 0.5 * np.cos(4 * np.pi * x + 1)
    du = torch.from_numpy(np.ascontiguousarray(u)).cuda()
    dd = torch.from_numpy(drifts).cuda()
    dtv = torch.from_numpy(tau * v).cuda()
    ks = [dev.build_kernel(n, tau, float(d)) for d in drifts]
    kt = torch.from_numpy(np.concatenate([k.window for k in ks])).cuda()
    fr = torch.tensor([k.first for k in ks], dtype=torch.int64, device="cuda")
    ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
    o = torch.empty_like(du)
    o1 = torch.empty_like(du)
    bl = torch.empty(lines, dtype=torch.int64, device="cuda")
    bl1 = torch.empty(lines, dtype=torch.int64, device="cuda")
    chained = api.FAST_CHAINED if seed % 2 else 0
    ok = True
    for step in range(6):
        dev.direct_f64(du, o1, kt, fr, tv=dtv, ktab_stride=2 * n + 1)
        dev.block_counts(du, bl1)
        dev.fast_f64(du, o, dd, tau, tv=dtv, blocks=bl, workspace=ws, flags=(api.FAST_STATS_VALID | chained) if step else 0)
        torch.cuda.synchronize()
        checks += 1
        if not torch.equal(o, o1) or not torch.equal(bl, bl1):
            fails += 1
            ok = False
            print("FAIL", seed, "step", step, "n", n, "lines", lines, "tau*n", tau * n, "tp", tp.tolist(),
                  "values", bool(torch.equal(o, o1)), "blocks", bool(torch.equal(bl, bl1)),
                  dev.fast_counters(ws, lines, n), flush=True)
            break
        du, o = o, du
    if ok and seed < 6:
        c = dev.fast_counters(ws, lines, n)
        print("seed", seed, "n", n, "tiles", c["tiles"], "direct gate/heavy", c["direct_tiles_gate"], c["direct_tiles_heavy"],
              "missed", c["missed_outputs"], flush=True)
print("done, checks:", checks, "failures:", fails)
