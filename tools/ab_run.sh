# Interleaved A/B timing of lib/ab/<name> builds: bash tools/ab_run.sh "<names>" <rounds> [quick_bench args]
names=$1; rounds=${2:-2}; shift 2
for r in $(seq $rounds); do
  for n in $names; do
    HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/$n/libhmx_gpu.so bash tools/quick_bench.sh "$@" > /dev/null 2>&1
    echo "== $n (round $r)"; python tools/show_bench.py
  done
done
