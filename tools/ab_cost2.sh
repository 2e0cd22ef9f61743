#!/bin/bash
# On the GPU box: 8-part balance of C5 (total) and C4 (per-vertex) under cost-model knobs.
for cfg in "TCB_COLD_COST=12" "TCB_COLD_COST=4" "TCB_COLD_COST=6 TCB_ITEM_COST=32" "TCB_COLD_COST=8 TCB_ITEM_COST=32 TCB_SEG_COST=2" "TCB_COLD_COST=4 TCB_ITEM_COST=16 TCB_WARP_COST=12"; do
  echo "== $cfg"
  env $cfg timeout 600 python tools/phase_probe.py --scale 26 --param 32 --pv 0 --iters 1 --parts 8 2>&1 | tail -1
  env $cfg timeout 300 python tools/phase_probe.py --pv 1 --iters 2 --parts 8 2>&1 | tail -1
done
