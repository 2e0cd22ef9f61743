#!/bin/bash
# On the GPU box: 8-part split balance under cost-model knobs (env), C4 per-vertex.
for cfg in ${COST_CFGS:-"TCB_COLD_COST=8 TCB_WARP_COST=12 TCB_ITEM_COST=64" "TCB_COLD_COST=16 TCB_WARP_COST=24 TCB_ITEM_COST=64" \
           "TCB_COLD_COST=12 TCB_WARP_COST=16 TCB_ITEM_COST=96 TCB_DENSE_COST=32" "TCB_COLD_COST=12 TCB_WARP_COST=16 TCB_ITEM_COST=64 TCB_DENSE_COST=64"}; do
  echo "== $cfg"; env $cfg python tools/phase_probe.py --iters 2 --parts 8 2>&1 | tail -1
done
