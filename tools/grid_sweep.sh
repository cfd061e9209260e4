#!/bin/bash
# co-located AMUSD: draft / verify SM split (AMUSD_FW_DRAFT_GRID), AMUSD engine only, no extras
for g in 48 56 64 72 80; do
  echo "DRAFT_GRID=$g $(AMUSD_FW_DRAFT_GRID=$g timeout 600 python bench.py --engines amusd --no-extras --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['amusd']['tokens_per_s'], d['amusd']['verify_steps'], d['amusd'].get('drafted'))")"
done
