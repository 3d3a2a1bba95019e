"""Seeded differential sweep of the multi-step / 2-D / relaxed paths against the reference library
(oracle/_ref): evolve (resident K2R and the launch loop, both engines), the 2-D split step (fast
layouts and direct), the host step, and the relaxed engine with eta > 0.  Random small sizes,
time steps across the anti-CFL range, drifts up to |tau P| = 4.  usage: fuzz_paths.py [seeds]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from tests import _oracle
from paper_1210_4090_b200 import api

dev = api.Device(0)
ref = _oracle.reference()
orc = _oracle.oracle()
nseeds = int(sys.argv[1]) if len(sys.argv) > 1 else 60
fails = 0
checks = 0


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def report(what, seed, **kw):
    global fails
    fails += 1
    print("FAIL", what, seed, kw, flush=True)


for seed in range(nseeds):
    rng = np.random.default_rng(20000 + seed)
    n = int(rng.choice([rng.integers(3, 40), rng.integers(40, 300), rng.integers(300, 1500)]))
    tau = 1.0 / (n * float(rng.uniform(0.05, 0.95)))
    tp = float(rng.uniform(-4, 4)) if rng.random() < 0.3 else float(rng.uniform(-1.5, 1.5))
    drift = tp / tau
    x = np.arange(n) / n
    u0 = np.sin(2 * np.pi * x) * rng.uniform(0.1, 2) + np.cumsum(rng.uniform(-1, 1, n)) / n * rng.uniform(0, 3)
    v = np.cos(2 * np.pi * x) * rng.uniform(0, 1.5) + rng.uniform(-0.3, 0.3, n)
    steps = int(rng.integers(1, 25))
    # ---- evolve: one line (resident) and a batch (launch loop when it fills the GPU; here still resident) ----
    try:
        uf, dr, bl, comp = ref.evolve(u0, tau, drift, v, steps, engine=1)
        for eng in (api.ENGINE_FAST, api.ENGINE_DIRECT):
            for resident in (1, 0):
                dev.set_evolve_resident(resident)
                du = t(u0[None, :].copy())
                sc = torch.empty_like(du)
                ws = torch.empty(dev.fast_workspace_bytes(1, n), dtype=torch.uint8, device="cuda")
                sd = torch.empty(steps, dtype=torch.float64, device="cuda")
                sb = torch.empty(steps, dtype=torch.int64, device="cuda")
                done = dev.evolve(du, sc, t(np.array([drift])), tau, steps, tv=t(tau * v), engine=eng, step_drift=sd,
                                  step_blocks=sb, workspace=ws)
                torch.cuda.synchronize()
                checks += 1
                if done != steps or not np.array_equal(du.cpu().numpy()[0], uf):
                    report("evolve state", seed, n=n, tau=tau, tp=tp, steps=steps, eng=eng, resident=resident)
                elif not np.array_equal(sb.cpu().numpy(), bl):
                    report("evolve blocks", seed, n=n, tau=tau, tp=tp, steps=steps, eng=eng, resident=resident)
                elif not np.allclose(sd.cpu().numpy(), dr, rtol=1e-11, atol=1e-13):
                    report("evolve drift", seed, n=n, tau=tau, tp=tp, steps=steps, eng=eng, resident=resident)
        dev.set_evolve_resident(1)
    except Exception as exc:
        report("evolve exception", seed, n=n, tau=tau, tp=tp, err=str(exc)[:200])
    # ---- host step, every engine (eta = 0 and eta > 0 for the relaxed one) ----
    try:
        lines = int(rng.integers(1, 12))
        U = np.stack([np.roll(u0, int(rng.integers(0, n))) * rng.uniform(0.5, 2) for _ in range(lines)])
        drifts = np.clip(rng.uniform(-1.5, 1.5, lines) / tau * (4 / 1.5 if rng.random() < 0.2 else 1), -1e3, 1e3)
        eta = float(rng.choice([0.0, 1e-7, 1e-4]))
        want0, wb0 = ref.step_lines(U, tau, drifts, v=v, eta=eta, engine=1, nthreads=4)
        want1, wb1 = ref.step_lines(U, tau, drifts, v=v, eta=eta, engine=0, nthreads=4)
        for eng, want, wb in ((api.ENGINE_FAST, want0, wb0), (api.ENGINE_DIRECT, want0, wb0), (api.ENGINE_RELAXED, want1, wb1)):
            blocks = np.empty(lines, np.int64)
            got = dev.step_host(U, drifts, tau, tv=tau * v, eta=eta, engine=eng, blocks=blocks)
            checks += 1
            if not np.array_equal(got, want):
                report("host step values", seed, n=n, tau=tau, eng=eng, eta=eta, lines=lines)
            elif not np.array_equal(blocks, wb):
                report("host step blocks", seed, n=n, tau=tau, eng=eng, eta=eta, lines=lines)
    except Exception as exc:
        report("host step exception", seed, n=n, tau=tau, err=str(exc)[:200])
    # ---- 2-D split step (n x n, n small): fast layouts and direct vs the reference ----
    try:
        m = int(rng.integers(3, 97))
        tau2 = 1.0 / (m * float(rng.uniform(0.05, 0.95)))
        d1, d2 = (rng.uniform(-3.5, 3.5, 2) if rng.random() < 0.3 else rng.uniform(-1.2, 1.2, 2)) / tau2
        u2 = rng.uniform(-1, 1, (m, m)) * rng.uniform(0.01, 1) + np.add.outer(np.sin(2 * np.pi * np.arange(m) / m),
                                                                              np.cos(2 * np.pi * np.arange(m) / m))
        want = ref.split_step_2d(u2, tau2, float(d1), float(d2), pot_kind=1, t=0.25)
        a = api.gen_cos(m)
        b = api.c4_time_term(0.25 + tau2)
        for eng, modes in ((api.ENGINE_DIRECT, (2,)), (api.ENGINE_FAST, (2, 0, 3, 5))):
            for mode in modes:
                dev.set_fast_line(mode)
                du = t(u2)
                o, tmp = torch.empty_like(du), torch.empty_like(du)
                ws = torch.empty(2 * dev.fast_workspace_bytes(m, m), dtype=torch.uint8, device="cuda")
                dev.split_step_2d(du, o, tmp, tau2, float(d1), float(d2), a1=t(a), a2=t(a), b=b, engine=eng, workspace=ws)
                torch.cuda.synchronize()
                checks += 1
                if not np.array_equal(o.cpu().numpy(), want):
                    report("split2d", seed, m=m, tau=tau2, d1=float(d1 * tau2), d2=float(d2 * tau2), eng=eng, mode=mode)
        dev.set_fast_line(2)
    except Exception as exc:
        dev.set_fast_line(2)
        report("split2d exception", seed, m=m, err=str(exc)[:200])
print("done, checks:", checks, "failures:", fails)
