mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32_order.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t_x.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_x.log
for ic in 4 8 12; do for w in 1.1 1.4 1.8; do echo "ITEM_COST=$ic HMX_ACC64_WEIGHT=$w"; HMX_CHAIN_ITEM_COST=$ic HMX_ACC64_WEIGHT=$w bash tools/quick_bench.sh --variants m1-mixed m2-single --steps 50; python tools/show_bench.py gpurun_out/qb.json 2>/dev/null | tail -2; done; done
