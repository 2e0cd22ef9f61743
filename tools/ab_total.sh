#!/bin/bash
# On the GPU box: C4 total-only whole count per library variant (main = the in-tree build).
for v in "$@"; do
  lib=variants/$v.so; [ "$v" = "main" ] && lib=paper_1909_02127_b200/libtcb200.so
  echo "== $v"; TCB200_LIB=$PWD/$lib python tools/phase_probe.py --pv 0 --iters 3 2>&1 | tail -1
done
