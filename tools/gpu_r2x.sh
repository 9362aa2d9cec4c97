mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32_order.py tests/test_gpu_parity.py tests/test_gpu_prepare.py -m gpu -x -q > gpurun_out/t_x.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_x.log
V="--variants m1-mixed m1-single m2-single"
echo "== stream small off"; HMX_STREAM_SMALL=0 bash tools/quick_bench.sh $V; python tools/show_bench.py gpurun_out/qb.json | tail -3
echo "== stream small on"; bash tools/quick_bench.sh $V; python tools/show_bench.py gpurun_out/qb.json | tail -3
for w in 1.0 1.8; do echo "== on, w=$w"; HMX_ACC64_WEIGHT=$w bash tools/quick_bench.sh $V; python tools/show_bench.py gpurun_out/qb.json | tail -3; done
for c in 3 5; do for ss in 0 1; do echo "== config $c stream_small=$ss"; HMX_STREAM_SMALL=$ss timeout 900 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --no-solve --variants m1-mixed m2-single > gpurun_out/qbc.json 2>/dev/null; python tools/show_bench.py gpurun_out/qbc.json | tail -2; done; done
