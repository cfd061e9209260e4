#!/bin/bash
# 1B draft: chain-phase (QKV / O) item sizes, solo and on the co-located 64 SMs.
run() { echo "$1 | $(env $1 timeout 60 python tools/fw_one.py --model 1b --iters 20 | cut -d' ' -f4-5) | $(env $1 timeout 60 python tools/fw_one.py --model 1b --iters 20 --grid 64 | cut -d' ' -f4-5)"; }
run "X=0"
run "AMUSD_FW_UNITS_O=4"
run "AMUSD_FW_UNITS_QKV=4"
run "AMUSD_FW_UNITS_QKV=4 AMUSD_FW_UNITS_O=4"
run "X=0"
