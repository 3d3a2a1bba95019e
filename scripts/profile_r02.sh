#!/bin/bash
# Round-2 profiles (run on the GPU box from the repo root; every ncu command runs only after the
# same command line exited 0 without ncu).  Reports land in gpurun_out/.
O=gpurun_out
# 1. K2 on C2: one launch after 1000 steps (the bench step: no block counts)
python scripts/prof_c2.py --pre 1000 > $O/p1.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fast_kernel -s 1003 -c 1 -f -o $O/r02_k2c2 \
    python scripts/prof_c2.py --pre 1000 > $O/ncu1.log 2>&1
# 2. the bench's launch list (share of each kernel in a step)
python bench.py --steps 2 --warmup 3 --presteps 3 --no-extras --no-cpu-baseline > $O/p2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --presteps 3 --no-extras --no-cpu-baseline > $O/ncu2.log 2>&1
# 3. the fused C4 split step: per-launch times, instructions, DRAM bytes (steps 5..8)
python scripts/prof_c4.py --steps 3 > $O/p3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -s 20 -c 8 --csv --log-file $O/r02_c4_launches.csv python scripts/prof_c4.py --steps 3 \
    > $O/ncu3.log 2>&1
# 4. the C4 transpose + statistics kernel and the second sweep in full
python scripts/prof_c4.py --steps 3 > $O/p4.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"transpose_stats|fast_kernel" -s 22 -c 2 -f \
    -o $O/r02_c4 python scripts/prof_c4.py --steps 3 > $O/ncu4.log 2>&1
# 5. K1 on C3: screened fp64 (default) and fp32 (FADD + FMNMX3)
python scripts/time_k1.py 1 > $O/p5.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"screen_kernel|direct_kernel" -c 6 -f \
    -o $O/r02_k1c3 python scripts/time_k1.py 1 > $O/ncu5.log 2>&1
ls -la $O
