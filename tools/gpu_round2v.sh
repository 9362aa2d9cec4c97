mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/t_all_v.log 2>&1; echo "tests rc=$?"; tail -40 gpurun_out/t_all_v.log | grep -E "passed|failed|error" 
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_v.log
timeout 600 python bench.py > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_v.json
