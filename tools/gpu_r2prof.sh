# round-2 profile captures: quick bench of every variant, plan notes, ncu --set full of the FP32-order stage 1 / stage 2 kernels
mkdir -p gpurun_out
bash tools/quick_bench.sh; python tools/show_bench.py gpurun_out/qb.json 2>/dev/null | tail -9
for s in m1-mixed m2-single m1-single; do
  HMX_PLAN_TIMING=1 python tools/profile_matvec.py --scheme $s --iters 1 > gpurun_out/pm_$s.log 2>&1 || exit 1
  grep -h "hmx_plan_create" gpurun_out/pm_$s.log | tail -1
  ncu --set full --import-source on --clock-control none -k regex:'seg_kernel|s1_exact' -s 2 -c 2 \
    -o gpurun_out/r2fifo_$s python tools/profile_matvec.py --scheme $s --iters 1 > gpurun_out/pr_$s.log 2>&1
done
ls gpurun_out | grep r2fifo
