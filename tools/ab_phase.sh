#!/bin/bash
# On the GPU box: phase timings of each variant: tools/ab_phase.sh pv name1 name2 ...
pv=$1; shift
for v in "$@"; do
  lib=variants/$v.so; [ "$v" = "main" ] && lib=paper_1909_02127_b200/libtcb200.so
  echo "== $v pv=$pv"; TCB200_LIB=$PWD/$lib python tools/phase_probe.py --pv $pv --iters 3 2>&1 | tail -14 | grep -E "join|rows|frontier|total|^[0-9]"
done
