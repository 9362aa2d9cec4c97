mkdir -p gpurun_out
for v in r1w8192 r2w8192 r1w16384 r2w16384 r1w4096; do
  HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/$v/libhmx_gpu.so timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve \
    --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_m_$v.json 2> gpurun_out/qb_m_$v.err; tail -1 gpurun_out/qb_m_$v.err
done
HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/r2w8192/libhmx_gpu.so timeout 600 python -m pytest tests/test_gpu_fp32_order.py -q > gpurun_out/t_m.log 2>&1; tail -2 gpurun_out/t_m.log
