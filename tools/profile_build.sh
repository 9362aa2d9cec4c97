# Launch list of the on-device H-matrix compression (GPU ACA + kernel-entry
# assembly + compaction) at config 4, after the same command exited 0 without ncu.
python tools/build_timing.py 4 > gpurun_out/pb_plain.log 2>&1 || exit 1
cat gpurun_out/pb_plain.log | tail -5
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
  --log-file gpurun_out/round1_build_launches_config4.csv python tools/build_timing.py 4 > gpurun_out/pb_ncu.log 2>&1
ls -la gpurun_out/round1_build_launches_config4.csv
