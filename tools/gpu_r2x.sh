mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32_order.py tests/test_gpu_parity.py tests/test_gpu_prepare.py -m gpu -x -q > gpurun_out/t_x.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_x.log
bash tools/quick_bench.sh --variants m1-single m1-mixed; python tools/show_bench.py gpurun_out/qb.json 2>/dev/null | tail -2
timeout 600 python bench.py --config 2 --steps 200 --warmup 10 --no-cpu-baseline --no-solve --variants m1-single m1-mixed > gpurun_out/qb2.json 2>/dev/null; python tools/show_bench.py gpurun_out/qb2.json | tail -2
