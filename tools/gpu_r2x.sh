mkdir -p gpurun_out
for c in 1 2 3; do
  HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/olds1/libhmx_gpu.so python tools/ab_bitwise.py --config $c --schemes m1-single --out gpurun_out/y_old.npz
  python tools/ab_bitwise.py --config $c --schemes m1-single --out gpurun_out/y_new.npz
  python -c "
import numpy as np
a=np.load('gpurun_out/y_old.npz'); b=np.load('gpurun_out/y_new.npz')
for k in a.files: print('config $c', k, 'bitwise equal:', np.array_equal(a[k], b[k]), float(np.max(np.abs(a[k]-b[k]))))
"
done
timeout 900 python -m pytest tests/test_gpu_fp32_order.py tests/test_gpu_parity.py tests/test_gpu_prepare.py -m gpu -x -q > gpurun_out/t_x.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_x.log
bash tools/quick_bench.sh --variants m1-single; python tools/show_bench.py gpurun_out/qb.json | tail -1
for c in 2 3; do timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --no-solve --variants m1-single > gpurun_out/qb3.json 2>/dev/null; python tools/show_bench.py gpurun_out/qb3.json | tail -1; done
