#!/bin/bash
# Round profiles (run on the GPU box from the repo root): K2 on C2, the bench launch list,
# and the widened rows' kernels.  Reports land in gpurun_out/.
set -x
O=gpurun_out
ncu --set full --import-source on --clock-control none -k regex:fast_kernel -s 1000 -c 1 -f -o $O/k2c2 \
    python scripts/prof_c2.py --pre 1000 > $O/ncu_k2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --presteps 3 --no-extras --no-cpu-baseline > $O/ncu_launch.log 2>&1
for k in tropical_gemm_kernel karp_cluster_kernel relaxed_scatter_kernel semidiscrete_kernel; do
  ncu --set full --clock-control none -k regex:$k -s 1 -c 1 -f -o $O/$k python scripts/prof_f234.py > $O/ncu_$k.log 2>&1
done
ls -la $O
