mkdir -p gpurun_out
for v in n3w8192 n4w6144 n2w8192 n3w12288 n4w8192; do
  HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/$v/libhmx_gpu.so timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve \
    --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_h_$v.json 2> gpurun_out/qb_h_$v.err; tail -1 gpurun_out/qb_h_$v.err
done
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_large.py::test_config5_sampled_rows > gpurun_out/t_h.log 2>&1; tail -6 gpurun_out/t_h.log
