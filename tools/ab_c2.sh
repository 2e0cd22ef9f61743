#!/bin/bash
# On the GPU box: C2 (ER) and C4 phases per library variant.
for v in "$@"; do
  lib=variants/$v.so; [ "$v" = "main" ] && lib=paper_1909_02127_b200/libtcb200.so
  echo "== $v"
  TCB200_LIB=$PWD/$lib python tools/phase_probe.py --kind er --scale 20 --param 32 --pv 0 --iters 3 2>&1 | tail -1
  TCB200_LIB=$PWD/$lib python tools/phase_probe.py --kind er --scale 20 --param 32 --pv 1 --iters 3 2>&1 | tail -1
  TCB200_LIB=$PWD/$lib python tools/phase_probe.py --iters 2 2>&1 | tail -1
done
