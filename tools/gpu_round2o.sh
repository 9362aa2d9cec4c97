mkdir -p gpurun_out
timeout 400 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_o.json 2> gpurun_out/qb_o.err; tail -1 gpurun_out/qb_o.err
timeout 2000 python -m pytest tests -m gpu -q --deselect tests/test_gpu_parity_large.py::test_config5_sampled_rows > gpurun_out/t_o.log 2>&1; tail -8 gpurun_out/t_o.log
