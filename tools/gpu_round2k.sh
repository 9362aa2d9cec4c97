mkdir -p gpurun_out
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_k.json 2> gpurun_out/qb_k.err; tail -1 gpurun_out/qb_k.err
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_parity_large.py::test_config5_sampled_rows > gpurun_out/t_k.log 2>&1; tail -12 gpurun_out/t_k.log
