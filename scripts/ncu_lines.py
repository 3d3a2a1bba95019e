"""Attribute ncu per-SASS instruction counts / stall samples to CUDA source
lines via nvdisasm line info.  usage: ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_SUBSTR"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kname = sys.argv[1:4]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
lines_of = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    cur_fn, cur_line = None, None
    for ln in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn and kname in cur_fn:
            lines_of[int(m.group(1), 16)] = cur_line
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ia, ie, ss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][ia], 16)
agg = collections.defaultdict(lambda: [0, 0])
for r in data:
    off = int(r[ia], 16) - base
    key = lines_of.get(off, "?")
    agg[key][0] += int(r[ie] or 0)
    agg[key][1] += int(r[ss] or 0)
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instr {ti}, stall samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"{k:22s} instr {v[0]/ti*100:5.1f}%  stalls {v[1]/ts*100:5.1f}%")
