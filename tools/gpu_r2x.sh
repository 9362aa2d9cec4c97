mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fp32_order.py tests/test_gpu_parity.py tests/test_gpu_prepare.py tests/test_gpu_distributed.py tests/test_gpu_reference_suite.py -m gpu -x -q > gpurun_out/t_x.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_x.log
bash tools/quick_bench.sh; python tools/show_bench.py gpurun_out/qb.json | tail -8
for c in 2 3; do timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m2-mixed m3:c=3 m1-single > gpurun_out/qb3.json 2>/dev/null; python tools/show_bench.py gpurun_out/qb3.json | tail -5; done
