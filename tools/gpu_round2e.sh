mkdir -p gpurun_out
export HMX_SHIM_LOGDIR=gpurun_out HMX_SHIM_WORKER_TIMEOUT=150 HMX_SHIM_TRACE=1 HMX_SHIM_WAIT_S=60
timeout 300 python -m pytest tests/test_gpu_dist_shim.py -q -x -k "2-auto" > gpurun_out/t_shim.log 2>&1; tail -3 gpurun_out/t_shim.log
unset HMX_SHIM_TRACE
timeout 300 python -m pytest tests/test_drop_in_refshape.py -q > gpurun_out/t_refshape.log 2>&1; tail -3 gpurun_out/t_refshape.log
