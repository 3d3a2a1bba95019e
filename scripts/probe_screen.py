"""Screened-K1 fallback rates and timings on C4 sweeps and C5 lines."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import api  # noqa: E402

dev = api.Device(0)


def timed(fn):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


res = {}
# C4 x2 sweep of u0 (rows), n = 2048, tau = 0.01, P = -0.7
n = 2048
u = torch.from_numpy(api.gen_c4_u0(n)).cuda()
for P in (0.3, -0.7):
    K = dev.build_kernel(n, 0.01, P)
    dk = torch.from_numpy(K.window).cuda()
    df = torch.full((n,), K.first, dtype=torch.int64, device="cuda")
    o = torch.empty_like(u)
    for mode, name in ((api.DIRECT_PLAIN, "plain"), (api.DIRECT_SCREENED, "screened")):
        dev.set_direct_mode(mode)
        dev.direct_f64(u, o, dk, df)
        dev.direct_stats(reset=True)
        ms = timed(lambda: dev.direct_f64(u, o, dk, df))
        res[f"c4_P{P}_{name}"] = {"ms": ms, **dev.direct_stats(), "outputs": n * n}
# C5 line
n = 1 << 20
u5 = torch.from_numpy(api.gen_c5_lines(0, 1, n)).cuda()
K = dev.build_kernel(n, 0.005, 0.25)
dk = torch.from_numpy(K.window).cuda()
df = torch.full((1,), K.first, dtype=torch.int64, device="cuda")
o = torch.empty_like(u5)
for mode, name in ((api.DIRECT_PLAIN, "plain"), (api.DIRECT_SCREENED, "screened")):
    dev.set_direct_mode(mode)
    dev.direct_stats(reset=True)
    ms = timed(lambda: dev.direct_f64(u5, o, dk, df))
    res[f"c5_{name}"] = {"ms": ms, **dev.direct_stats(), "outputs": n}
print(json.dumps(res))
