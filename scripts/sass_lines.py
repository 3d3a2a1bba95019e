"""Static SASS instruction counts per source line of one kernel (nvdisasm -g output).
usage: python scripts/sass_lines.py FILE.sass KERNEL_SUBSTR [file.cu] [lo hi]"""
import re
import sys
from collections import Counter, defaultdict

path, sub = sys.argv[1], sys.argv[2]
src = sys.argv[3] if len(sys.argv) > 3 else "fast.cu"
lo, hi = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (0, 1 << 30)
cur, inside, line = None, False, None
per = Counter()
ops = defaultdict(Counter)
for ln in open(path):
    if ln.startswith("//---------------------") and ".text." in ln:
        inside = sub in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
    if m and line:
        if line[0] == src and lo <= line[1] <= hi:
            per[line[1]] += 1
            ops[line[1]][m.group(2).split(".")[0]] += 1
for l in sorted(per):
    print(l, per[l], dict(ops[l].most_common(6)))
print("total", sum(per.values()))
