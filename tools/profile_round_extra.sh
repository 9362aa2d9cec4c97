bash tools/profile_round.sh round1f > gpurun_out/prof.log 2>&1
# ncu of m1-single and m2-single stage 2 too
for s in m1-single m2-single; do
  f=$(echo $s | tr -d ':=')
  ncu --set full --import-source on --clock-control none -k regex:seg_kernel -s 2 -c 2 \
    -o gpurun_out/round1f_$f python tools/profile_matvec.py --scheme $s --iters 1 > gpurun_out/pr_$f.log 2>&1
done
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
ls gpurun_out
