#!/bin/bash
# On the GPU box: whole-count C4 phase timings (pv and total-only) per variant:
#   tools/ab_c4.sh name1 name2 ...   (main = the in-tree build)
for v in "$@"; do
  lib=variants/$v.so; [ "$v" = "main" ] && lib=paper_1909_02127_b200/libtcb200.so
  for pv in 1 0; do
    echo "== $v pv=$pv"; TCB200_LIB=$PWD/$lib python tools/phase_probe.py --pv $pv --iters 2 2>&1 | tail -1
  done
done
