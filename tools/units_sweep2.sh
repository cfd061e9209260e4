#!/bin/bash
# persistent forward item sizes: 1B (all SMs / the co-located 64) and 8B (all / the co-located 84)
run() { echo "$1 | 1b $(env $1 timeout 60 python tools/gv_probe.py --models 1b --grids 0,64 --rows 1 --paths persistent --iters 20 2>/dev/null | python -c "import sys,json; print(' '.join(str(json.loads(l)['ms']) for l in sys.stdin))") | 8b $(env $1 timeout 90 python tools/gv_probe.py --models 8b --grids 0,84 --rows 1,4 --paths persistent --iters 10 2>/dev/null | python -c "import sys,json; print(' '.join(str(json.loads(l)['ms']) for l in sys.stdin))")"; }
run "X=0"
run "AMUSD_FW_UNITS_O=4"
run "AMUSD_FW_UNITS_O=4 AMUSD_FW_UNITS_QKV=4"
run "AMUSD_FW_UNITS_GU=32"
run "AMUSD_FW_UNITS_GU=32 AMUSD_FW_UNITS_O=4 AMUSD_FW_UNITS_QKV=4"
run "X=0"
