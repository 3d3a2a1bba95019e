"""Stall-reason breakdown per CUDA source line (ncu source page + nvdisasm line info).
usage: ncu_stalls_by_line.py REPORT LIB KERNEL_SUBSTR SRC_FILE [first_line last_line]"""
import collections, csv, glob, io, os, re, subprocess, sys, tempfile
rep, lib, kname, srcf = sys.argv[1:5]
rng = (int(sys.argv[5]), int(sys.argv[6])) if len(sys.argv) > 6 else None
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
lines_of = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    fn = ln_ = None
    for ln in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m: fn = m.group(1); continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m: ln_ = (os.path.basename(m.group(1)), int(m.group(2))); continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and fn and kname in fn: lines_of[int(m.group(1), 16)] = ln_
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ia = hdr.index("Address"); ie = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
agg = collections.defaultdict(lambda: collections.Counter())
for r in data:
    key = lines_of.get(int(r[ia], 16) - base)
    if not key: continue
    c = agg[key]
    c["instr"] += int(r[ie] or 0)
    for i in stall_cols:
        c[hdr[i]] += int(r[i] or 0)
src = open(srcf).read().splitlines()
tot = sum(sum(v for k, v in c.items() if k.startswith("stall")) for c in agg.values()) or 1
items = sorted(agg.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k.startswith("stall")))
for (f, l), c in items[:30]:
    if rng and f == os.path.basename(srcf) and not (rng[0] <= l <= rng[1]): continue
    st = sum(v for k, v in c.items() if k.startswith("stall"))
    top = ", ".join(f"{k[6:]}:{v*100//max(st,1)}%" for k, v in c.most_common() if k.startswith("stall") and v * 10 >= st)
    text = src[l - 1].strip()[:70] if f == os.path.basename(srcf) else f
    print(f"{st/tot*100:5.1f}% {f}:{l:<4d} {text:70s} | {top}")
