#!/bin/bash
# Full GPU check: smoke + pytest -m gpu + bench (+ optional ncu) on one box.
mkdir -p gpurun_out
./tools/gpu_tests.sh
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
