mkdir -p gpurun_out
rm -f gpurun_out/mem_trace5.txt
( while true; do free -g | awk '/Mem/{print $3}' >> gpurun_out/mem_trace5.txt; sleep 2; done ) &
MON=$!
timeout 1500 python -m pytest "tests/test_gpu_parity_large.py::test_config5_sampled_rows" -q -s > gpurun_out/t_large5.log 2>&1; tail -3 gpurun_out/t_large5.log
kill $MON
sort -n gpurun_out/mem_trace5.txt | tail -1
