# round-2 GPU check: FP32 order tests, the multi-process dist path, bench, full suite
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fp32_order.py tests/test_gpu_dist_shim.py -q -m gpu -x > gpurun_out/t_new.log 2>&1; tail -3 gpurun_out/t_new.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -2 gpurun_out/bench_c4.err
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/t_gpu_all.log 2>&1; tail -8 gpurun_out/t_gpu_all.log
