"""Hot SASS regions of one kernel in an ncu report (source page, per-instruction execution counts).
usage: python scripts/ncu_hot.py REPORT [launch_skip] [--dump lo-hi ...]"""
import csv
import io
import subprocess
import sys
import collections

rep = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 0
dumps = [tuple(int(x, 16) for x in a.split("-")) for a in sys.argv[3:] if "-" in a and not a.startswith("--")]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", str(skip),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
print(rows[0][1][:90])
h = rows[1]
d = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name" and d:
        break
    if len(r) == len(h) and r[0].startswith("0x"):
        d.append(r)
ia, ie, isrc, iss = h.index("Address"), h.index("Instructions Executed"), h.index("Source"), h.index(
    "Warp Stall Sampling (All Samples)")
hot = [(int(r[ia], 16), int(r[ie] or 0), int(r[iss] or 0), r[isrc]) for r in d]
base = hot[0][0]
tot = sum(x[1] for x in hot)
stot = sum(x[2] for x in hot) or 1
print("total warp instr", tot, "sass", len(hot), "stall samples", stot)
if dumps:
    for lo, hi in dumps:
        for a, e, s, src in hot:
            if lo <= a - base <= hi and e > 0:
                print(f"{a-base:6x} {e:9d} {s:5d} {src}")
    sys.exit(0)
reg, cur = [], None
for a, e, s, src in hot:
    if e > 0:
        if cur and a - cur[1] <= 0x20:
            cur[1] = a
            cur[2] += e
            cur[3] += s
        else:
            if cur:
                reg.append(cur)
            cur = [a, a, e, s]
reg.append(cur)
for r in sorted(reg, key=lambda r: -r[2])[:16]:
    print(f"{r[0]-base:6x}-{r[1]-base:6x} n={(r[1]-r[0])//16+1:4d} instr={r[2]:10d} {r[2]/tot*100:5.1f}%  stall {r[3]/stot*100:5.1f}%")
c = collections.Counter()
for a, e, s, src in hot:
    c[e] += e
print("by execution count:", [(e, round(v / tot * 100, 1)) for e, v in sorted(c.items(), key=lambda kv: -kv[1])[:10]])
