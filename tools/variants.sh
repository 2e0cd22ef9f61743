#!/bin/bash
# Build A/B variants of libtcb200.so here: tools/variants.sh name "-DFLAGS" [name "-DFLAGS" ...]
set -e
ROOT=$(cd $(dirname $0)/.. && pwd)
mkdir -p $ROOT/variants
while [ $# -gt 1 ]; do
  make -s -C $ROOT/paper_1909_02127_b200/csrc OBJDIR=$ROOT/build/obj_$1 OUT=$ROOT/variants/$1.so EXTRA_NVFLAGS="$2" -j8 2>&1 | grep -E "error|spill" || true
  shift 2
done
