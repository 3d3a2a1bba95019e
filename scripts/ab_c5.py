"""A/B timing of the C5 K2 run (64 x 2^20, 200 chained steps from the seeded u0) for several
builds of the library, each in a fresh process.  usage: python scripts/ab_c5.py LIB.so [LIB2.so ...]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, torch, time
sys.path.insert(0, __ROOT__)
from paper_1210_4090_b200 import _capi, api
_capi.LIB_PATH = __LIB__
_capi.load(required_symbols={k for k in _capi.SIGNATURES if k.startswith(("lob_ctx", "lob_last", "lob_version",
    "lob_fast", "lob_minplus_fast", "lob_launch", "lob_gen", "lob_kernel_mech"))})
n, lines, tau, p = 1 << 20, 64, 0.005, 0.25
dev = api.Device(0)
a0 = torch.from_numpy(api.gen_c5_lines(0, lines, n)).cuda()
tv = torch.from_numpy(api.tau_v(api.gen_potential(3, n), tau)).cuda()
dr = torch.full((lines,), p, dtype=torch.float64, device="cuda")
ws = torch.empty(dev.fast_workspace_bytes(lines, n), dtype=torch.uint8, device="cuda")
bl = torch.empty(lines, dtype=torch.int64, device="cuda")
res = []
for rep in range(3):
    a = a0.clone(); b = torch.empty_like(a)
    torch.cuda.synchronize()
    seg = []
    for k in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(50 * k, 50 * (k + 1)):
            dev.fast_f64(a, b, dr, tau, tv=tv, blocks=bl, workspace=ws,
                         flags=api.FAST_CHAINED | (api.FAST_STATS_VALID if i else 0))
            a, b = b, a
        e1.record(); torch.cuda.synchronize()
        seg.append(round(e0.elapsed_time(e1) / 50, 4))
    res.append(seg)
print(json.dumps({"lib": __LIB__, "ms_per_step_by_50": res}))
'''
for lib in sys.argv[1:]:
    code = CHILD.replace("__ROOT__", repr(ROOT)).replace("__LIB__", repr(os.path.abspath(lib)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-2000:], flush=True)
