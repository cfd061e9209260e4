#!/bin/bash
# ncu evidence for profiles/: launch list of eager verify+draft forwards, and a
# full capture of the dominant kernel (verify gate/up tcgen05 GEMM).
mkdir -p gpurun_out
K='regex:k_gemm_tc|k_gemv|k_attention|k_embed|k_argmax_final'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches.csv python tools/ncu_forward.py > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 200 -c 4 -o gpurun_out/prof_gemm -f python tools/ncu_forward.py > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 700 -c 5 -o gpurun_out/prof_gemv -f python tools/ncu_forward.py > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/ncu_launch.log gpurun_out/ncu_full.log gpurun_out/ncu_full2.log
