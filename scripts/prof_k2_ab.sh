O=gpurun_out
python scripts/prof_c2.py --pre 1000 > $O/p1.log 2>&1 && \
LOB_LIB=paper_1210_4090_b200/build_old/liblaxol_b200.so ncu --set full --import-source on --clock-control none -k regex:fast_kernel -s 1003 -c 1 -f -o $O/k2old \
    python scripts/prof_c2.py --pre 1000 > $O/ncu_old.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fast_kernel -s 1003 -c 1 -f -o $O/k2new \
    python scripts/prof_c2.py --pre 1000 > $O/ncu_new.log 2>&1
ls -la $O
