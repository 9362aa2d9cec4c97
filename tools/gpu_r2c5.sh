# config-5 bench line (two level-8 spheres, N = 2,621,440) with the round-2 kernels
mkdir -p gpurun_out
timeout 2400 python bench.py --config 5 --steps 30 --warmup 3 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m2-mixed m3:c=3 > gpurun_out/bench_config5.json 2> gpurun_out/bench_config5.err; echo "rc=$?"
python tools/show_bench.py gpurun_out/bench_config5.json | tail -5; tail -3 gpurun_out/bench_config5.err
