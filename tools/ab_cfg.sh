# A/B of builds at configs 2, 3 and 4: bash tools/ab_cfg.sh "<names>" <rounds> [variants...]
names=$1; rounds=${2:-2}; shift 2
for r in $(seq $rounds); do
  for n in $names; do
    for c in 2 3; do
      echo "== $n config $c (round $r)"
      HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/$n/libhmx_gpu.so python tools/plan_info.py --config $c --variants "$@" 2>&1 | cut -c1-60
    done
    echo "== $n config 4 (round $r)"
    HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/$n/libhmx_gpu.so bash tools/quick_bench.sh --variants "$@" > /dev/null 2>&1; python tools/show_bench.py
  done
done
