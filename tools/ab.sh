#!/bin/bash
# A/B timing of variant libraries on C4: tools/ab.sh pv name1 name2 ...
pv=$1; shift
for v in "$@"; do
  lib=variants/$v.so; [ "$v" = "main" ] && lib=paper_1909_02127_b200/libtcb200.so
  echo -n "$v pv=$pv: "; TCB200_LIB=$PWD/$lib python tools/prof_count.py --iters 3 --pv $pv | tail -1 | cut -c1-80
done
