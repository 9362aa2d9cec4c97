# quick matvec-only timing of every variant at config 4 (no solve, no CPU leg)
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-solve \
  --variants m1-double m1-mixed m2-mixed m3:c=3 m3:c=-1 m1-single m2-single m2-double "$@" \
  > gpurun_out/qb.json 2> gpurun_out/qb.err; tail -2 gpurun_out/qb.err
