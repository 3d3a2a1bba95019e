"""Long-run golden fixtures from the reference itself (oracle/_ref), run in the
build container where /root/reference is present (a few minutes on 8 cores):

    python tests/golden/make_golden_long.py

* c2_hbar_n1024.npz — the C2 H-bar sweep downscaled in N only (SURVEY.md 8d,
  "C2 CPU slice"): the 256 C2 drifts, C2 potential, tau=0.02, u0=0, 5000
  steps at N=1024, reference evolve (ConvEngine::Naive) per line; H-bar(P)
  for all 256 lines, final state + per-step drift/blocks for 5 lines.
* c5_n16384.npz — C5's spectrum / kinetics / potential at N=2^14 (2 lines,
  seeds 5000, 5001), 40 steps of reference evolve.
* c4_n128.npz — C4 (P=(0.3,-0.7), V=cos cos + 0.2 sin(2 pi t)) at 128^2,
  20 reference split_step_nd steps from u0 = sin(2 pi x1) + cos(2 pi x2).
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_1210_4090_b200 import api  # noqa: E402  (input generators only)
from tests import _oracle  # noqa: E402

ref = _oracle.reference()
assert ref is not None, "needs oracle/_ref (make -f oracle/Makefile ref)"
POOL = ThreadPoolExecutor(os.cpu_count() or 1)


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, {k: getattr(v, "shape", v) for k, v in arrays.items()}, flush=True)


# 1. C2 H-bar sweep at N=1024
n, tau, steps = 1024, 0.02, 5000
drifts = api.gen_c2_drifts(256)
v = api.gen_potential(2, n)
u0 = np.zeros(n)
res = list(POOL.map(lambda p: ref.evolve(u0, tau, float(p), v, steps, engine=1), drifts))
hbar = np.array([np.sum(r[0] - u0) / n / (steps * tau) for r in res])
keep = np.array([0, 37, 128, 200, 255])
save("c2_hbar_n1024.npz", drifts=drifts, v=v, hbar=hbar, keep=keep,
     u_final=np.stack([res[i][0] for i in keep]), step_drift=np.stack([res[i][1] for i in keep]),
     step_blocks=np.stack([res[i][2] for i in keep]))

# 2. C5 spectrum at N=2^14, 2 lines, 40 steps
n5, tau5, steps5 = 1 << 14, 0.005, 40
u5 = api.gen_c5_lines(0, 2, n5)
v5 = api.gen_potential(3, n5)
res = list(POOL.map(lambda l: ref.evolve(u5[l], tau5, 0.25, v5, steps5, engine=1), range(2)))
save("c5_n16384.npz", u0=u5, v=v5, u_final=np.stack([r[0] for r in res]),
     step_drift=np.stack([r[1] for r in res]), step_blocks=np.stack([r[2] for r in res]))

# 3. C4 at 128^2, 20 split steps
n4, tau4, steps4 = 128, 0.01, 20
u = api.gen_c4_u0(n4)
states = []
for s in range(steps4):
    u = ref.split_step_2d(u, tau4, 0.3, -0.7, pot_kind=1, t=s * tau4)
    if s in (0, 1, 4, 19):
        states.append(u.copy())
save("c4_n128.npz", u0=api.gen_c4_u0(n4), states=np.stack(states), at=np.array([0, 1, 4, 19]))
