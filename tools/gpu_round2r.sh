mkdir -p gpurun_out
(cat /sys/fs/cgroup/memory.max; free -g) > gpurun_out/mem_info.txt 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m2-single > gpurun_out/qb_r.json 2> gpurun_out/qb_r.err; tail -1 gpurun_out/qb_r.err
( while true; do free -g | awk '/Mem/{print $3}' >> gpurun_out/mem_trace.txt; sleep 2; done ) &
MON=$!
timeout 900 python -m pytest "tests/test_gpu_parity_large.py::test_full_products_every_scheme" -q > gpurun_out/t_large34.log 2>&1; tail -3 gpurun_out/t_large34.log
timeout 900 python -m pytest "tests/test_gpu_parity_large.py::test_config5_sampled_rows" -q -s > gpurun_out/t_large5.log 2>&1; tail -3 gpurun_out/t_large5.log
kill $MON
