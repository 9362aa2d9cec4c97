mkdir -p gpurun_out
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_t.json 2> gpurun_out/qb_t.err; tail -1 gpurun_out/qb_t.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:seg_kernel -s 1 -c 1 \
    -o gpurun_out/r2t_m1mixed_s2 python tools/profile_matvec.py --scheme m1-mixed --iters 1 > gpurun_out/ncu_t1.log 2>&1; tail -1 gpurun_out/ncu_t1.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"seg_kernel|s1_exact" -c 2 \
    -o gpurun_out/r2t_m1single python tools/profile_matvec.py --scheme m1-single --iters 1 > gpurun_out/ncu_t2.log 2>&1; tail -1 gpurun_out/ncu_t2.log
