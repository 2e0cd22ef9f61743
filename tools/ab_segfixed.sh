#!/bin/bash
# On the GPU box: 8-part maxima (C4 total / per-vertex, C5 total) per TCB_SEG_FIXED value.
# (TCB_SEG_FIXED was a temporary PivotCost knob for this sweep; not adopted, removed: profiles/README.md)
for f in "$@"; do
  echo "== seg_fixed=$f"
  TCB_SEG_FIXED=$f python tools/phase_probe.py --pv 0 --iters 2 --parts 8 2>&1 | grep "parts=" | tail -1
  TCB_SEG_FIXED=$f python tools/phase_probe.py --pv 1 --iters 2 --parts 8 2>&1 | grep "parts=" | tail -1
  TCB_SEG_FIXED=$f python tools/phase_probe.py --scale 26 --param 32 --pv 0 --iters 2 --parts 8 2>&1 | grep "parts=" | tail -1
done
