mkdir -p gpurun_out
export HMX_SHIM_LOGDIR=gpurun_out HMX_SHIM_WORKER_TIMEOUT=150
timeout 400 python -m pytest tests/test_gpu_dist_shim.py -q -x -k "2-auto" > gpurun_out/t_shim.log 2>&1; tail -3 gpurun_out/t_shim.log
for v in minb4 minb3; do
  HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/$v/libhmx_gpu.so timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve \
    --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_$v.json 2> gpurun_out/qb_$v.err; tail -1 gpurun_out/qb_$v.err
done
timeout 300 python -m pytest tests/test_gpu_fp32_order.py tests/test_drop_in_refshape.py -q > gpurun_out/t_fp32b.log 2>&1; tail -3 gpurun_out/t_fp32b.log
