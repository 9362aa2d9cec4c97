# round-2 records: bench lines at configs 2 and 3 (every variant), launch list of the default bench command
mkdir -p gpurun_out
for c in 2 3; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 10 --variants m1-double m1-mixed m2-mixed m3:c=3 m3:c=-1 m1-single m2-single \
    > gpurun_out/bench_config$c.json 2> gpurun_out/bench_config$c.err; echo "config $c rc=$?"
  python tools/show_bench.py gpurun_out/bench_config$c.json | tail -8
done
python bench.py --steps 3 --warmup 3 --variants m1-double m1-mixed --no-cpu-baseline --no-solve > gpurun_out/ll_plain.json 2> gpurun_out/ll_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/round2_launches.csv \
  python bench.py --steps 3 --warmup 3 --variants m1-double m1-mixed --no-cpu-baseline --no-solve > gpurun_out/ll.log 2>&1
tail -3 gpurun_out/round2_launches.csv | cut -c1-200
