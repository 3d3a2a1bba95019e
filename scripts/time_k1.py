"""K1 on C3 (4096 x 4096, tau=0.01, P=0): screened vs plain fp64 and fp32 (CUDA events, median of reps)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import _capi, api  # noqa: E402
import os  # noqa: E402

if os.environ.get("LOB_LIB"):
    _capi.LIB_PATH = os.path.abspath(os.environ["LOB_LIB"])

dev = api.Device(0)
n = lines = 4096
K = dev.build_kernel(n, 0.01, 0.0)
u = torch.from_numpy(api.gen_c3_lines(0, lines, n)).cuda()
o = torch.empty_like(u)
dk = torch.from_numpy(K.window).cuda()
df = torch.full((lines,), K.first, dtype=torch.int64, device="cuda")
cand = lines * n * (2 * n + 1)


def med(fn, reps=int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    fn()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


res = {}
for name, mode in (("screened", api.DIRECT_SCREENED), ("plain", api.DIRECT_PLAIN)):
    dev.set_direct_mode(mode)
    dev.direct_stats(reset=True)
    t = med(lambda: dev.direct_f64(u, o, dk, df))
    res[name] = {"ms": t, "cand_per_s": cand / t * 1e3, **dev.direct_stats()}
    res[name]["out_sum"] = float(o.sum())
dev.set_direct_mode(api.DIRECT_SCREENED)
u32, o32, dk32 = u.float(), torch.empty_like(u, dtype=torch.float32), dk.float()
t = med(lambda: dev.direct_f32(u32, o32, dk32, df))
res["fp32"] = {"ms": t, "cand_per_s": cand / t * 1e3}
print(json.dumps(res))
