mkdir -p gpurun_out
python tools/profile_matvec.py --scheme m1-mixed --iters 1 > gpurun_out/pm.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:seg_kernel -s 1 -c 1 \
    -o gpurun_out/r2_m1mixed_s2_win python tools/profile_matvec.py --scheme m1-mixed --iters 1 > gpurun_out/ncu_m1mixed.log 2>&1; tail -1 gpurun_out/ncu_m1mixed.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:s1_exact -c 1 \
    -o gpurun_out/r2_m1single_s1 python tools/profile_matvec.py --scheme m1-single --iters 1 > gpurun_out/ncu_m1single.log 2>&1; tail -1 gpurun_out/ncu_m1single.log
