#!/bin/bash
# Work-item size sweep (AMUSD_FW_UNITS_<KIND>, 16 KB weight units per item), solo launches:
# 8B verify (1 and 4 rows) and 1B draft on all SMs.
run() { echo "$1 | $(env $1 timeout 60 python tools/fw_one.py --iters 10 | cut -d' ' -f4-5) | $(env $1 timeout 60 python tools/fw_one.py --iters 10 --rows 4 | cut -d' ' -f4-5) | $(env $1 timeout 60 python tools/fw_one.py --model 1b --iters 20 | cut -d' ' -f4-5)"; }
run "X=0"
for u in 16; do run "AMUSD_FW_UNITS_QKV=$u"; done
for u in 4 16; do run "AMUSD_FW_UNITS_O=$u"; done
for u in 8 32; do run "AMUSD_FW_UNITS_GU=$u"; done
for u in 8 32; do run "AMUSD_FW_UNITS_DOWN=$u"; done
run "X=0"
