mkdir -p gpurun_out
python tools/profile_matvec.py --scheme m1-single --iters 1 > gpurun_out/pm.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:seg_kernel -s 0 -c 1 \
    -o gpurun_out/r2_m1single_s2 python tools/profile_matvec.py --scheme m1-single --iters 1 > gpurun_out/ncu_a.log 2>&1; tail -1 gpurun_out/ncu_a.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:s1_exact -c 1 \
    -o gpurun_out/r2_m1single_s1b python tools/profile_matvec.py --scheme m1-single --iters 1 > gpurun_out/ncu_b.log 2>&1; tail -1 gpurun_out/ncu_b.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve --variants m1-double m1-single > gpurun_out/qb_n.json 2> gpurun_out/qb_n.err; tail -1 gpurun_out/qb_n.err
