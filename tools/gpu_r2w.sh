# exact-order FP32 stage 2: quick bench of every variant + ncu --set full of m1-mixed / m1-single / m2-single stage 2
mkdir -p gpurun_out
bash tools/quick_bench.sh; python tools/show_bench.py gpurun_out/qb.json 2>/dev/null | tail -30
for s in m1-mixed m2-single m1-single; do
  python tools/profile_matvec.py --scheme $s --iters 1 > gpurun_out/pm_$s.log 2>&1 || exit 1
  ncu --set full --import-source on --clock-control none -k regex:seg_kernel -s 2 -c 2 \
    -o gpurun_out/r2w_$s python tools/profile_matvec.py --scheme $s --iters 1 > gpurun_out/pr_$s.log 2>&1
done
ls -la gpurun_out
