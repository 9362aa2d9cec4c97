mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32_order.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t_x.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_x.log
for w in 0.8 1.0; do echo "HMX_ACC64_WEIGHT=$w"; HMX_ACC64_WEIGHT=$w bash tools/quick_bench.sh --variants m1-mixed m1-single m2-single; python tools/show_bench.py gpurun_out/qb.json 2>/dev/null | tail -3; done
s=m1-mixed
ncu --set full --import-source on --clock-control none -k regex:seg_kernel -s 3 -c 1 \
    -o gpurun_out/r2z_$s python tools/profile_matvec.py --scheme $s --iters 1 > gpurun_out/pr_$s.log 2>&1
