# Launch lists of one BiCG-STAB solve (m1-double, configs 4 and 2) for the
# per-kernel share of the solve.  ncu cannot list kernel nodes of a graph with
# a conditional node, so the lists use the stream path (HMX_SOLVER_NO_GRAPH:
# the same kernels, bitwise-identical results) plus one whole-graph capture.
for c in 4 2; do
  python tools/profile_solve.py --config $c --scheme m1-double > gpurun_out/ps_plain_$c.log 2>&1 || exit 1
  HMX_SOLVER_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/round1_solver_launches_config$c.csv \
    python tools/profile_solve.py --config $c --scheme m1-double > gpurun_out/ps_ncu_$c.log 2>&1
  ncu --graph-profiling graph --metrics gpu__time_duration.sum --clock-control none -c 50 --csv \
    --log-file gpurun_out/round1_solver_graph_config$c.csv \
    python tools/profile_solve.py --config $c --scheme m1-double > gpurun_out/ps_graph_$c.log 2>&1
done
ls -la gpurun_out/round1_solver_*
