"""Generate tests/golden/*.npz from the reference itself (oracle/_ref, the
laxol library compiled from /root/reference/proj/src) — run in the build
container where the reference is present:  python tests/golden/make_golden.py
Fixtures are small; every vector is produced by the reference's own API."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_1210_4090_b200 import api  # noqa: E402  (input generators only)
from tests import _oracle  # noqa: E402

ref = _oracle.reference()
assert ref is not None, "needs oracle/_ref (make -f oracle/Makefile ref)"


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, {k: getattr(v, "shape", v) for k, v in arrays.items()})


# 1. kernel windows (build_kernel) for small shapes + the C1/C3/C4 windows
ks = {}
for (n, tau, p) in [(24, 0.25, 0.4), (100, 0.1, 0.0), (600, 0.04, 1.0), (1024, 0.05, 0.5), (4096, 0.01, 0.0),
                    (2048, 0.01, 0.3), (2048, 0.01, -0.7)]:
    w, first, arg, st = ref.kernel(n, tau, p)
    ks[f"w_{n}_{tau}_{p}"] = w
    ks[f"meta_{n}_{tau}_{p}"] = np.array([first, arg], np.int64)
save("kernels.npz", **ks)

# 2. kinetic_convolve (Naive) on seeded random periodic lines, drifts {0,.4,-.7,1}
rng = np.random.default_rng(39)
kc = {}
for drift in (0.0, 0.4, -0.7, 1.0):
    u = rng.uniform(-1, 1, 24)
    out, blocks, _ = ref.kinetic_convolve(u, 24, 0.25, drift, engine=1)
    kc[f"u_{drift}"] = u
    kc[f"out_{drift}"] = out
    kc[f"blocks_{drift}"] = np.array([blocks])
save("kinetic_convolve_n24.npz", **kc)

# 3. C1 in full: N=1024, tau=0.05, P=0.5, V=cos(2 pi x), u0=sin(2 pi x), 2000 steps
n, tau, steps = 1024, 0.05, 2000
u0 = api.gen_sin(n)
v = api.gen_potential(1, n)
uf, drift, blocks, comp = ref.evolve(u0, tau, 0.5, v, steps, engine=1)
hbar = np.sum(uf - u0) / n / (steps * tau)
save("c1_evolve.npz", u0=u0, v=v, u_final=uf, step_drift=drift, step_blocks=blocks,
     hbar=np.array([hbar]), completed=np.array([comp]))
print("C1 H-bar = mean(u_T - u_0)/T =", repr(hbar))

# 4. C3 lines 0..3, one step (N=4096, tau=0.01, P=0, V=0)
u = api.gen_c3_lines(0, 4, 4096)
out, blk = ref.step_lines(u, 0.01, 0.0, v=None, engine=1, nthreads=4)
save("c3_lines0-3.npz", u=u, out=out, blocks=blk)

# 5. C2-shaped short run at N=2048 (per-line P, C2 potential), 5 steps from 0, 4 lines
n2, tau2 = 2048, 0.02
drifts = api.gen_c2_drifts(256)[[0, 85, 170, 255]]
v2 = api.gen_potential(2, n2)
u = np.zeros((4, n2))
hist = []
for s in range(5):
    u, blk = ref.step_lines(u, tau2, drifts, v=v2, t=s * tau2, engine=1, nthreads=4)
    hist.append(u.copy())
save("c2_n2048_5steps.npz", drifts=drifts, v=v2, states=np.stack(hist))

# 6. 2-D split steps (16x16 brute-force-pinned, and C4's potential at 32x32)
rng = np.random.default_rng(42)
u16 = rng.uniform(-1, 1, (16, 16))
o16 = ref.split_step_2d(u16, 0.25, 0.0, 0.5)
u32 = api.gen_c4_u0(32)
o32 = ref.split_step_2d(u32, 0.05, 0.3, -0.7, pot_kind=1, t=0.35)
save("split2d.npz", u16=u16, out16=o16, u32=u32, out32=o32)

# 7. decomposition block counts (KAT cosine + random walks, eta 0 / 1e-3 / 0.5)
rng = np.random.default_rng(19)
vs = [rng.uniform(-1, 1, int(rng.integers(2, 200))) for _ in range(50)]
counts = np.array([[ref.decompose(x, eta)[0] for eta in (0.0, 1e-3, 0.5)] for x in vs])
lens = np.array([len(x) for x in vs])
save("decompose.npz", values=np.concatenate(vs), lens=lens, counts=counts)
