mkdir -p gpurun_out
export HMX_SHIM_LOGDIR=gpurun_out HMX_SHIM_WORKER_TIMEOUT=150 HMX_SHIM_TRACE=1 HMX_SHIM_WAIT_S=60
timeout 300 python -m pytest tests/test_gpu_dist_shim.py -q -x -k "2-auto" > gpurun_out/t_shim.log 2>&1; tail -3 gpurun_out/t_shim.log
unset HMX_SHIM_TRACE
python tools/profile_matvec.py --scheme m1-mixed --iters 1 > gpurun_out/pm.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:seg_kernel -s 1 -c 1 \
    -o gpurun_out/r2_m1mixed_s2 python tools/profile_matvec.py --scheme m1-mixed --iters 1 > gpurun_out/ncu_m1mixed.log 2>&1; tail -2 gpurun_out/ncu_m1mixed.log
timeout 300 python -m pytest tests/test_drop_in_refshape.py -q > gpurun_out/t_refshape.log 2>&1; tail -3 gpurun_out/t_refshape.log
