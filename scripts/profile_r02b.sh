#!/bin/bash
# Round-2 (later session) measurements on the GPU box, from the repo root.  Every ncu command
# runs only after the same command exited 0 without ncu.  Outputs in gpurun_out/.
O=gpurun_out
python bench.py > $O/bench.json 2> $O/bench.err
# bench launch list (share of each kernel in a step)
python bench.py --steps 2 --warmup 3 --presteps 3 --no-extras --no-cpu-baseline > $O/p2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --presteps 3 --no-extras --no-cpu-baseline > $O/ncu2.log 2>&1
# the C4 split step (transposes + K2L row sweeps): per-launch time, instructions, L2 bytes
python scripts/time_c4.py --steps 10 --mode 2 > $O/p3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --cache-control none --clock-control none -k regex:"line_kernel|transpose" -s 20 -c 8 --csv \
    --log-file $O/r02_c4_k2l_launches.csv python scripts/time_c4.py --steps 10 --mode 2 > $O/ncu3.log 2>&1
# K2 on C2 (bench step), full set with source
python scripts/prof_c2.py --pre 1000 > $O/p1.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fast_kernel -s 1003 -c 1 -f -o $O/r02_k2c2 \
    python scripts/prof_c2.py --pre 1000 > $O/ncu1.log 2>&1
# the K2L row sweep of C4 in full
ncu --set full --import-source on --clock-control none -k regex:line_kernel -s 21 -c 1 -f -o $O/r02_k2l_c4 \
    python scripts/time_c4.py --steps 10 --mode 2 > $O/ncu4.log 2>&1
ls -la $O
