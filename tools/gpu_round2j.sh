mkdir -p gpurun_out
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_j.json 2> gpurun_out/qb_j.err; tail -1 gpurun_out/qb_j.err
timeout 900 python -m pytest tests/test_gpu_fp32_order.py tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_drop_in_refshape.py -q > gpurun_out/t_j.log 2>&1; tail -6 gpurun_out/t_j.log
