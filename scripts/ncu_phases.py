"""Attribute ncu per-SASS instruction counts / stall samples of one kernel to
its OUTERMOST source line inside the kernel (nvdisasm -gi inline chains), then
to named line ranges.  usage: ncu_phases.py REPORT CUBIN KERNEL_SUBSTR SRC_BASENAME RANGES
RANGES = name:lo-hi,name:lo-hi,...  (lines of SRC_BASENAME)"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, kname, srcbase, ranges = sys.argv[1:6]
rng = [(r.split(":")[0], *map(int, r.split(":")[1].split("-"))) for r in ranges.split(",")]
dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
line_of, ops = {}, {}
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
        cur = (outer[0] if __import__("os").environ.get("INNER") else outer[-1]) if outer else None
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", ln)
    if m and cur_fn and kname in cur_fn:
        line_of[int(m.group(1), 16)] = cur
        ops[int(m.group(1), 16)] = m.group(2).strip()
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ia, ie, ss, isrc = (hdr.index("Address"), hdr.index("Instructions Executed"),
                    hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"))
base = int(data[0][ia], 16)
agg = collections.defaultdict(lambda: [0, 0])
mism = 0
for r in data:
    off = int(r[ia], 16) - base
    l = line_of.get(off)
    if off in ops and ops[off].split()[0].lstrip("@!P0123456789T ") not in r[isrc]:
        mism += 1
    name = "?"
    if l is not None:
        for nm, lo, hi in rng:
            if lo <= l <= hi:
                name = nm
                break
        else:
            name = f"line{l}"
    agg[name][0] += int(r[ie] or 0)
    agg[name][1] += int(r[ss] or 0)
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instr {ti}, stall samples {ts}, opcode mismatches {mism}/{len(data)}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(__import__("os").environ.get("TOPN", "30"))]:
    print(f"{k:22s} instr {v[0]/ti*100:5.1f}%  stalls {v[1]/ts*100:5.1f}%")
