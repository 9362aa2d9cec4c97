mkdir -p gpurun_out
timeout 400 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_p.json 2> gpurun_out/qb_p.err; tail -1 gpurun_out/qb_p.err
timeout 600 python -m pytest tests/test_gpu_fp32_order.py tests/test_gpu_parity.py -q > gpurun_out/t_p.log 2>&1; tail -3 gpurun_out/t_p.log
