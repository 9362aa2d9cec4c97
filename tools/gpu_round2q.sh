mkdir -p gpurun_out
for wt in 0.5 1.0 2.0; do
  HMX_ACC64_WEIGHT=$wt timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m2-single > gpurun_out/qb_q_$wt.json 2> gpurun_out/qb_q_$wt.err; tail -1 gpurun_out/qb_q_$wt.err
done
for v in em3 em3w12; do
  HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/$v/libhmx_gpu.so timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_q_$v.json 2> gpurun_out/qb_q_$v.err; tail -1 gpurun_out/qb_q_$v.err
done
timeout 900 python -m pytest tests/test_gpu_parity_large.py -q -m "gpu" > gpurun_out/t_large.log 2>&1; tail -4 gpurun_out/t_large.log
