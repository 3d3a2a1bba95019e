"""Summarise an ncu report (SOL, occupancy, issue, hot SASS regions)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keep = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Theoretical Occupancy", "SM Frequency")
for row in csv.DictReader(io.StringIO(out)):
    if row.get("Metric Name") in keep:
        print(f'{row["Kernel Name"][:30]:30s} {row["Metric Name"]:40s} {row["Metric Value"]} {row["Metric Unit"]}')
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
if len(rows) > 2:
    hdr = rows[0]
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                 "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "smsp__inst_executed_pipe_fp64.sum", "gpu__time_duration.sum"):
        if name in hdr:
            i = hdr.index(name)
            print(f"{name:60s} {rows[2][i]} {rows[1][i]}")
if len(sys.argv) > 2:
    s = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                       capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(s)))
    hdr, data = rows[1], rows[2:]
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[ie] or 0) for r in data)
    st = sum(int(r[ss] or 0) for r in data) or 1
    print("total warp instructions", tot)
    W = int(sys.argv[2])
    agg = {}
    for i, r in enumerate(data):
        k = i // W
        a = agg.setdefault(k, [0, 0])
        a[0] += int(r[ie] or 0)
        a[1] += int(r[ss] or 0)
    for k, (a, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
        print(f"sass[{k*W:5d}..] instr {a/tot*100:5.1f}%  stall-samples {b/st*100:5.1f}%  first: {data[k*W][1].strip()[:60]}")
