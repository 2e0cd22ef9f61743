#!/bin/bash
# On the GPU box: whole-count and 8-part phase timings of each variant:
#   tools/ab_phase8.sh pv name1 name2 ...   (main = the in-tree build)
pv=$1; shift
for v in "$@"; do
  lib=variants/$v.so; [ "$v" = "main" ] && lib=paper_1909_02127_b200/libtcb200.so
  echo "== $v pv=$pv"; TCB200_LIB=$PWD/$lib python tools/phase_probe.py --pv $pv --iters 2 2>&1 | tail -14 | grep -E "join|rows|total|^[0-9]"
  TCB200_LIB=$PWD/$lib python tools/phase_probe.py --pv $pv --iters 2 --parts 8 2>&1 | tail -1
done
