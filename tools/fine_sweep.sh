#!/bin/bash
# per-kind fine-grained dependencies (AMUSD_FW_FINE = bitmask of consumer kinds:
# 1 QKV, 2 attention, 4 O, 8 gate/up, 16 down, 64 LM head)
run() { echo "$1 | 1b $(env $1 timeout 60 python tools/gv_probe.py --models 1b --grids 0,64 --rows 1 --paths persistent --iters 20 2>/dev/null | python -c "import sys,json; print(' '.join(str(json.loads(l)['ms']) for l in sys.stdin))") | 8b $(env $1 timeout 90 python tools/gv_probe.py --models 8b --grids 0,84 --rows 1,4 --paths persistent --iters 10 2>/dev/null | python -c "import sys,json; print(' '.join(str(json.loads(l)['ms']) for l in sys.stdin))")"; }
for v in 0 1 2 4 8 16 64 24 80 127 0; do run "AMUSD_FW_FINE=$v"; done
