#!/bin/bash
# On the GPU box: 8-part balance of C5 (total) and C4 (per-vertex) vs the small-bin cost multiplier.
for cfg in ${COST_CFGS:-"TCB_SLAB_COST=6"}; do
  echo "== $cfg"
  env $cfg timeout 600 python tools/phase_probe.py --scale 26 --param 32 --pv 0 --iters 2 --parts 8 2>&1 | tail -1
  env $cfg timeout 300 python tools/phase_probe.py --pv 1 --iters 2 --parts 8 2>&1 | tail -1
done
