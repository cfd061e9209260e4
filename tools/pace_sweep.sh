#!/bin/bash
# AMUSD verify pacing (AMUSD_VERIFY_MIN_WINDOW / AMUSD_VERIFY_WAIT_US), co-located 1B + 8B
for mw in "1 0" "2 1000" "3 1500" "3 3000" "4 2500" "4 4000" "6 5000"; do
  set -- $mw
  echo "MIN_WINDOW=$1 WAIT_US=$2 $(AMUSD_VERIFY_MIN_WINDOW=$1 AMUSD_VERIFY_WAIT_US=$2 timeout 600 python bench.py --engines amusd --no-extras --no-cpu-baseline --steps 3 --warmup 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); a=d['amusd']; print(a['tokens_per_s'], a['verify_steps'], a['rollbacks'], a['drafted'])")"
done
