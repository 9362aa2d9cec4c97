mkdir -p gpurun_out
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_l.json 2> gpurun_out/qb_l.err; tail -1 gpurun_out/qb_l.err
timeout 900 python -m pytest tests/test_gpu_fp32_order.py tests/test_gpu_solver_envelope.py tests/test_gpu_parity.py -q -x > gpurun_out/t_l.log 2>&1; tail -4 gpurun_out/t_l.log
timeout 1200 python tools/stagnation_check.py --level 8 --spheres 1 --iters 30 --part gpu --out gpurun_out/stag_gpu.json > gpurun_out/stag_gpu.log 2>&1; tail -2 gpurun_out/stag_gpu.log
