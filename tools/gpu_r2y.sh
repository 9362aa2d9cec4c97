mkdir -p gpurun_out
for s in m1-mixed m1-single; do
  python tools/profile_matvec.py --scheme $s --iters 1 > gpurun_out/pm_$s.log 2>&1 || exit 1
  ncu --set full --import-source on --clock-control none -k regex:seg_kernel -s 3 -c 1 \
    -o gpurun_out/r2y_$s python tools/profile_matvec.py --scheme $s --iters 1 > gpurun_out/pr_$s.log 2>&1
done
ls -la gpurun_out | tail -5
