mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fp32_order.py tests/test_drop_in_refshape.py tests/test_gpu_dist_shim.py tests/test_gpu_parity.py -q -x > gpurun_out/t_f.log 2>&1; tail -4 gpurun_out/t_f.log
for v in w8m4 w8m3 w6m4 w12m3; do
  for wt in 2.5 1.0; do
  HMX_ACC64_WEIGHT=$wt HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/$v/libhmx_gpu.so timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve \
    --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_${v}_$wt.json 2> gpurun_out/qb_${v}_$wt.err; tail -1 gpurun_out/qb_${v}_$wt.err
  done
done
