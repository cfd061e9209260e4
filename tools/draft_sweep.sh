#!/bin/bash
# 1B draft forward (1 row) under the persistent-forward knobs: L2 prefetch window, next-layer
# prefetch, two CTAs per SM (grid 296, shallow rings).
run() { echo -n "$1 :: "; shift; env "$@" timeout 60 python tools/fw_one.py --model 1b --iters 30 --pos 300 2>&1 | tail -1; }
run base A=1
for mb in 8 16 32 64 96; do run "l2 ${mb}MB" AMUSD_FW_L2_MB=$mb; done
run "prefetch_next" AMUSD_FW_PREFETCH_NEXT=1
for st in 2 3 4 5 6; do run "stages $st" AMUSD_FW_STAGES=$st; done
for st in 2 3; do echo -n "grid296 stages $st :: "; AMUSD_FW_STAGES=$st timeout 60 python tools/fw_one.py --model 1b --iters 30 --pos 300 --grid 296 2>&1 | tail -1; done
for u in 8 32; do run "units $u" AMUSD_FW_UNITS=$u; done
