set -x
mkdir -p gpurun_out
(lscpu; nproc; free -g; nvidia-smi) > gpurun_out/box_info.txt 2>&1
timeout 300 python tools/sgemv_order_probe.py 24 --json gpurun_out/sgemv_box.json > gpurun_out/sgemv_box.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_fp32_order.py -q -m gpu > gpurun_out/t_fp32.log 2>&1; tail -3 gpurun_out/t_fp32.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -3 gpurun_out/bench_c4.err
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/t_gpu_all.log 2>&1; tail -15 gpurun_out/t_gpu_all.log
