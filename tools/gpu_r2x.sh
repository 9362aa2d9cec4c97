mkdir -p gpurun_out
V="--variants m1-mixed m1-single m2-single"
for n in nb3 nb3pair nb4pair nb3 nb3pair; do
export HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/$n/libhmx_gpu.so
echo "== $n"; bash tools/quick_bench.sh $V; python tools/show_bench.py gpurun_out/qb.json | tail -3
done
