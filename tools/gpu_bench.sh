#!/bin/bash
# Bench + launch list + dominant-kernel ncu capture on the GPU box.
mkdir -p gpurun_out
timeout 300 python bench.py --shapes tiny --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tiny.json 2> gpurun_out/bench_tiny.err
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gemv|k_attention|k_embed|k_argmax_final|k_draft|k_verify|k_hash" -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --profile-only --new-tokens 16 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gemvILi16E.*Li2ELi1E" -s 40 -c 1 -o gpurun_out/prof_gateup -f python bench.py --profile-only --new-tokens 16 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gemvILi2E.*Li2ELi1E" -s 40 -c 1 -o gpurun_out/prof_draft_gateup -f python bench.py --profile-only --new-tokens 16 > gpurun_out/ncu_full2.log 2>&1
tail -3 gpurun_out/bench_tiny.err; cat gpurun_out/bench_tiny.json; tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/ncu_full.log
