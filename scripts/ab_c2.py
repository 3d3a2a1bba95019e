"""A/B timing of the C2 K2 step for several builds of the library.
usage: python scripts/ab_c2.py LIB.so [LIB2.so ...]   (each timed in a fresh process)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, torch
sys.path.insert(0, __ROOT__)
from paper_1210_4090_b200 import _capi, api
_capi.LIB_PATH = __LIB__
n, tau, L = 65536, 0.02, 256
dev = api.Device(0)
dr = torch.from_numpy(api.gen_c2_drifts(L)).cuda()
tv = torch.from_numpy(api.tau_v(api.gen_potential(2, n), tau)).cuda()
x = torch.zeros((L, n), dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
ws = torch.empty(dev.fast_workspace_bytes(L, n), dtype=torch.uint8, device="cuda")
bl = torch.empty(L, dtype=torch.int64, device="cuda")
CH = getattr(api, "FAST_CHAINED", 0) if __CHAINED__ else 0
def run(k, i0):
    global x, y
    for i in range(k):
        dev.fast_f64(x, y, dr, tau, tv=tv, blocks=None if __NOB__ else bl, workspace=ws,
                     flags=CH | (api.FAST_STATS_VALID if i0 + i else 0))
        x, y = y, x
run(1000, 0)
res = []
for r in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    run(50, 1)
    e1.record(); torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 50)
print(json.dumps({"lib": __LIB__, "chained": __CHAINED__, "ms": sorted(res)}))
'''
for lib in sys.argv[1:]:
    chained = ":chained" in lib
    nob = ":nob" in lib
    lib = lib.split(":")[0]
    code = CHILD.replace("__ROOT__", repr(ROOT)).replace("__LIB__", repr(os.path.abspath(lib)))
    code = code.replace("__CHAINED__", repr(chained)).replace("__NOB__", repr(nob))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-2000:], flush=True)
