# ncu --set full of one stage-1 and one stage-2 launch per headline scheme at
# BASELINE configs 2 and 3 (config 3: "matvec-only throughput sweep with ncu
# HBM GB/s").  Usage (under gpurun): bash tools/profile_configs.sh
for c in 3 2; do
  for s in m1-double m1-mixed m2-mixed m3:c=3; do
    f=$(echo $s | tr -d ':=')
    python tools/profile_matvec.py --config $c --scheme $s --iters 1 > /dev/null 2>&1 || exit 1
    ncu --set full --clock-control none -k regex:seg_kernel -s 2 -c 2 \
      -o gpurun_out/round1c${c}_$f python tools/profile_matvec.py --config $c --scheme $s --iters 1 \
      > gpurun_out/pc_${c}_$f.log 2>&1
  done
done
ls gpurun_out/round1c*
