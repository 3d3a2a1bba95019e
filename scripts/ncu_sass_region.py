"""Print SASS with executed-instruction counts for one source-line range of a
kernel (outermost inlined line).  usage: ncu_sass_region.py REPORT CUBIN KERNEL SRC LO HI"""
import csv
import io
import re
import subprocess
import sys

rep, cubin, kname, srcbase, lo, hi = sys.argv[1:7]
lo, hi = int(lo), int(hi)
dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
line_of = {}
cur_fn, cur = None, None
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', ln)
    if m:
        chain = [(m.group(1), int(m.group(2)))] + [(f, int(l)) for f, l in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3))]
        outer = [l for f, l in chain if f.endswith(srcbase)]
        cur = outer[-1] if outer else None
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", ln)
    if m and cur_fn and kname in cur_fn:
        line_of[int(m.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ia, ie, ss, isrc = (hdr.index("Address"), hdr.index("Instructions Executed"),
                    hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"))
base = int(data[0][ia], 16)
tot = 0
for r in data:
    off = int(r[ia], 16) - base
    l = line_of.get(off)
    if l is not None and lo <= l <= hi:
        n = int(r[ie] or 0)
        tot += n
        if n:
            print(f"{off:05x} L{l:<4d} {n:>9d} {int(r[ss] or 0):>5d}  {r[isrc]}")
print("total", tot)
