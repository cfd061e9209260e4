#!/bin/bash
# dependency-poll back-off (AMUSD_POLL_NS, compile time): prebuilt variants in variants/
for v in 100 25 50 200 100; do
  cp variants/libamusd_poll$v.so paper_2410_17375_b200/libamusd.so
  echo "POLL_NS=$v | 1b $(timeout 60 python tools/gv_probe.py --models 1b --grids 0,64 --rows 1 --paths persistent --iters 20 2>/dev/null | python -c "import sys,json; print(' '.join(str(json.loads(l)['ms']) for l in sys.stdin))") | 8b $(timeout 90 python tools/gv_probe.py --models 8b --grids 0,84 --rows 1,4 --paths persistent --iters 10 2>/dev/null | python -c "import sys,json; print(' '.join(str(json.loads(l)['ms']) for l in sys.stdin))")"
done
