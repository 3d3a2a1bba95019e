"""Write the round's ncu summaries into profiles/ from reports in gpurun_out/.
usage: python scripts/write_profiles.py TAG K2_REPORT K1S_REPORT K1P_REPORT K3_REPORT"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, k2, k1s, k1p, k3 = sys.argv[1:6]
LIB = os.path.join(ROOT, "paper_1210_4090_b200", "lib", "liblaxol_b200.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, capture_output=True)


def run(*args):
    return subprocess.run([sys.executable, *args], capture_output=True, text=True, cwd=ROOT).stdout


def src_line(path, pat):
    for i, l in enumerate(open(os.path.join(ROOT, path)).read().splitlines(), 1):
        if pat in l:
            return i
    raise SystemExit(f"pattern not found: {pat}")


F = "paper_1210_4090_b200/csrc/fast.cu"
k = src_line(F, "fast_kernel(")
w0 = src_line(F, "// ---- warp 0: line gate")
b1 = src_line(F, "__syncthreads();  // keys, LUT, gate")
pc = src_line(F, "process_chunk<true>(S, ca);")
pf = src_line(F, "process_chunk<false>(S, ca);")
ep = src_line(F, "// ---- epilogue: exact min")
ts = src_line(F, "tile_stats<true>(vals, Tl, j0, line, tile, p, b, S.epi(), g_fsm_lut2);") - 1
ranges = (f"init:{k}-{w0 - 1},warp0_gate_scan_tma:{w0}-{b1},chunk_setup:{b1 + 1}-{pc - 1},emit_staged:{pc}-{pc},"
          f"emit_unstaged:{pf}-{pf},epilogue:{ep}-{ts - 1},tile_stats:{ts}-{ts + 3},blocks_tail:{ts + 4}-{ts + 30}")
with open(os.path.join(ROOT, "profiles", f"{tag}_k2_fast_c2_ncu_summary.txt"), "w") as f:
    f.write("# K2 fast_kernel, C2 (256 x 65536) after 1000 steps; one launch, ncu --set full --clock-control none\n")
    f.write(run("scripts/ncu_summary.py", k2))
    f.write("\n# instructions / stall samples by kernel phase (outermost source line; scripts/ncu_phases.py)\n")
    f.write(run("scripts/ncu_phases.py", k2, os.path.join(tmp, "fast.sm_100a.cubin"), "fast_kernelILb1ELb0ELb0E", "fast.cu",
                ranges))
with open(os.path.join(ROOT, "profiles", f"{tag}_k1_screen_c3_ncu_summary.txt"), "w") as f:
    f.write("# K1 screened (fp32 screen + fp64 span pass), C3 4096 x 4096 fp64, one launch\n")
    f.write(run("scripts/ncu_summary.py", k1s))
with open(os.path.join(ROOT, "profiles", f"{tag}_k1_direct_c3_ncu_summary.txt"), "w") as f:
    f.write("# K1 plain fp64 (LOB_DIRECT_PLAIN), C3 4096 x 4096, one launch\n")
    f.write(run("scripts/ncu_summary.py", k1p))
with open(os.path.join(ROOT, "profiles", f"{tag}_k3_split_c4_ncu_summary.txt"), "w") as f:
    f.write("# K3 + K2 sweeps of one C4 split step (2048^2): transpose, K2 sweep, potential, transpose, K2 sweep\n")
    f.write(run("scripts/ncu_summary.py", k3))
    f.write(subprocess.run(["ncu", "-i", k3, "--page", "raw", "--csv", "--metrics",
                            "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"],
                           capture_output=True, text=True).stdout)
print("ok")
