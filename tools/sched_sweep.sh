#!/bin/bash
B="python bench.py --no-extras --steps 2 --warmup 1 --engines amusd"
for cfg in "AMUSD_STREAM_PRIO=verify_high" "AMUSD_STREAM_PRIO=equal" "AMUSD_STREAM_PRIO=draft_high" "AMUSD_STREAM_PRIO=equal AMUSD_NO_PDL=1" "AMUSD_STREAM_PRIO=equal AMUSD_TC_GRID=120" "AMUSD_STREAM_PRIO=draft_high AMUSD_TC_GRID=128" "AMUSD_STREAM_PRIO=equal LEAD=4" "AMUSD_STREAM_PRIO=draft_high LEAD=8"; do
  L=$(echo $cfg | grep -o "LEAD=[0-9]*" | cut -d= -f2); E=$(echo $cfg | sed 's/LEAD=[0-9]*//')
  out=$(env $E $B ${L:+--lead $L} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); a=d['amusd']; print(round(a['tokens_per_s'],1), 'tok/s verify_steps', a['verify_steps'], 'drafted', a['drafted'])")
  echo "$cfg -> $out"
done
