#!/bin/bash
# On the GPU box: warm edge-list build time per library variant.
for v in "$@"; do
  lib=variants/$v.so; [ "$v" = "main" ] && lib=paper_1909_02127_b200/libtcb200.so
  echo "== $v"; TCB200_LIB=$PWD/$lib TCB_PHASES=0 python tools/build_probe.py 24 2>&1 | grep "^build"
done
