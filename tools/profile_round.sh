# Round profile captures (B200): launch list of the bench command and
# ncu --set full of one stage-1 + one stage-2 launch per headline scheme.
# Usage (under gpurun): bash tools/profile_round.sh <tag>
tag=${1:-round}
python bench.py --steps 3 --warmup 3 --variants m1-double --no-cpu-baseline --no-solve > gpurun_out/pr_plain.json 2> gpurun_out/pr_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 3 --warmup 3 --variants m1-double --no-cpu-baseline --no-solve > gpurun_out/pr_ll.log 2>&1
for s in m1-double m1-mixed m2-mixed m3:c=3; do
  python tools/profile_matvec.py --scheme $s --iters 1 > /dev/null 2>&1 || exit 1
  f=$(echo $s | tr -d ':=')
  ncu --set full --import-source on --clock-control none -k regex:seg_kernel -s 2 -c 2 \
    -o gpurun_out/${tag}_$f python tools/profile_matvec.py --scheme $s --iters 1 > gpurun_out/pr_$f.log 2>&1
done
ls gpurun_out/${tag}_*
