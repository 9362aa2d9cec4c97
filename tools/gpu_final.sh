# end-of-round validation and records: all GPU tests, smoke, default bench line, bench lines at configs 2-3, quick bench, ncu of the FP32-order kernels
mkdir -p gpurun_out
bash tools/gpu_full.sh
for c in 2 3; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 10 --variants m1-double m1-mixed m2-mixed m3:c=3 m3:c=-1 m1-single m2-single \
    > gpurun_out/bench_config$c.json 2> gpurun_out/bench_config$c.err; echo "config $c rc=$?"
  python tools/show_bench.py gpurun_out/bench_config$c.json | tail -7
done
bash tools/gpu_r2prof.sh
