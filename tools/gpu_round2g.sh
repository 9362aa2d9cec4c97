mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32_order.py tests/test_gpu_dist_shim.py tests/test_gpu_parity.py tests/test_gpu_acceptance.py -q > gpurun_out/t_g.log 2>&1; tail -6 gpurun_out/t_g.log
for wt in 2.5 1.0 0.5; do
  HMX_ACC64_WEIGHT=$wt timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve \
    --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_g_$wt.json 2> gpurun_out/qb_g_$wt.err; tail -1 gpurun_out/qb_g_$wt.err
done
