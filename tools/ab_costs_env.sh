#!/bin/bash
# On the GPU box: 8-part maxima (C4 per-vertex, C4 total, C5 total) per cost-model env setting:
#   tools/ab_costs_env.sh "TCB_WARP_COST=12" "TCB_WARP_COST=12 TCB_SMALL_COST=7" ...
for e in "$@"; do
  echo "== $e"
  env $e python tools/phase_probe.py --pv 1 --iters 2 --parts 8 2>&1 | grep "parts=" | tail -1
  env $e python tools/phase_probe.py --pv 0 --iters 2 --parts 8 2>&1 | grep "parts=" | tail -1
  env $e python tools/phase_probe.py --scale 26 --param 32 --pv 0 --iters 2 --parts 8 2>&1 | grep "parts=" | tail -1
done
