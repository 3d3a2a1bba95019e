"""e2e diagnostics: lob_step_host_f64 time vs raw pinned copies of the same bytes."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1210_4090_b200 import _capi, api  # noqa: E402
import os  # noqa: E402

if os.environ.get("LOB_LIB"):
    _capi.LIB_PATH = os.path.abspath(os.environ["LOB_LIB"])

L, N, TAU = 256, 65536, 0.02
dev = api.Device(0)
uh = torch.zeros((L, N), dtype=torch.float64, pin_memory=True)
oh = torch.empty_like(uh, pin_memory=True)
un, on = uh.numpy(), oh.numpy()
dh = api.gen_c2_drifts(L)
tvh = api.tau_v(api.gen_potential(2, N), TAU)
bh = np.empty(L, np.int64)
res = {"pinned": bool(uh.is_pinned())}
for lines in (256, 8):
    dev.step_host(un[:lines], dh[:lines], TAU, tv=tvh, out=on[:lines])
    t0 = time.perf_counter()
    for _ in range(5):
        dev.step_host(un[:lines], dh[:lines], TAU, tv=tvh, out=on[:lines])
    res[f"step_host_ms_{lines}"] = (time.perf_counter() - t0) / 5 * 1e3
d = torch.empty((L, N), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    d.copy_(uh, non_blocking=True)
    oh.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
res["raw_serial_ms"] = (time.perf_counter() - t0) / 5 * 1e3
print(json.dumps(res))
