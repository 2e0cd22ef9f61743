#!/bin/bash
# On the GPU box: C4 per-vertex 8-part maxima per cost-model env setting.
for e in "$@"; do
  echo "== $e"
  env $e python tools/phase_probe.py --pv 1 --iters 2 --parts 8 2>&1 | grep "parts=" | tail -1
done
