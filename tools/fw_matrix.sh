#!/bin/bash
# Persistent-forward timing matrix: 8B rows x context, 1B draft (one eager forward each, averaged).
for pos in 300 540; do for rows in 1 3 5; do timeout 60 python tools/fw_one.py --pos $pos --rows $rows --iters 10 | sed "s/^/pos=$pos /"; done; done
timeout 60 python tools/fw_one.py --model 1b --iters 20 | sed "s/^/pos=300 /"
timeout 60 python tools/fw_one.py --model 1b --pos 540 --iters 20 | sed "s/^/pos=540 /"
