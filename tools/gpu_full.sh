# full GPU validation: every -m gpu test, smoke(), the default bench line
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"; tail -25 gpurun_out/t_all.log | grep -E "passed|failed|error|Error" 
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_default.json
