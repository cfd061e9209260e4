#!/bin/bash
# Work-item size combos (AMUSD_FW_UNITS_<KIND>, 16 KB weight units per item) at the co-located
# SM shares: 8B verify (3 rows) on 84 SMs, 1B draft on 64 SMs.
run() { echo "$1 | $(env $1 timeout 60 python tools/fw_one.py --iters 10 --rows 3 --grid 84 | cut -d' ' -f4-5) | $(env $1 timeout 60 python tools/fw_one.py --model 1b --iters 20 --grid 64 | cut -d' ' -f4-5)"; }
run "X=0"
run "X=0"
run "AMUSD_FW_UNITS_GU=32 AMUSD_FW_UNITS_DOWN=32"
run "AMUSD_FW_UNITS_GU=32 AMUSD_FW_UNITS_DOWN=32 AMUSD_FW_UNITS_QKV=16 AMUSD_FW_UNITS_O=16"
run "AMUSD_FW_UNITS_GU=64 AMUSD_FW_UNITS_DOWN=64 AMUSD_FW_UNITS_QKV=16 AMUSD_FW_UNITS_O=16"
run "AMUSD_FW_UNITS_GU=32 AMUSD_FW_UNITS_DOWN=32 AMUSD_FW_UNITS_QKV=16"
