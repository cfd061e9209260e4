#!/bin/bash
# ncu evidence for profiles/ (run under gpurun; summarise here with
#   python tools/prof_summary.py <tag> gpurun_out/launches.csv gpurun_out/full.ncu-rep):
# launch list of the eager verify + draft forwards (the persistent k_forward; kernels
# inside graphs with conditional nodes cannot be profiled), one --set full capture of
# a verify forward and one of a draft forward.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python tools/ncu_forward.py > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward -s 5 -c 1 \
  -o gpurun_out/full -f python tools/ncu_forward.py > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward -s 7 -c 1 \
  -o gpurun_out/full_draft -f python tools/ncu_forward.py > gpurun_out/ncu_full_draft.log 2>&1
tail -n 2 gpurun_out/ncu_launch.log gpurun_out/ncu_full.log gpurun_out/ncu_full_draft.log
