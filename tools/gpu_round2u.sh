mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fp32_order.py -x -q > gpurun_out/t_u.log 2>&1; tail -2 gpurun_out/t_u.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-solve --variants m1-double m1-mixed m1-single m2-single > gpurun_out/qb_u.json 2> gpurun_out/qb_u.err; tail -1 gpurun_out/qb_u.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/qb_u.json').read().strip().splitlines()[-1])
for k,v in d.get('variants',{}).items(): print(k, v['ms'])
PY
