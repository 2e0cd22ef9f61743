#!/bin/bash
# Build an A/B variant of libtcb200.so with extra nvcc flags into build/variants/<name>.so
# usage: tools/build_variant.sh name "-DTCB_HOT_WIN=4 -DTCB_MIN_BLOCKS=3"
set -e
name=$1; flags=$2
ROOT=$(cd $(dirname $0)/.. && pwd)
mkdir -p $ROOT/variants
make -s -C $ROOT/paper_1909_02127_b200/csrc OBJDIR=$ROOT/build/obj_$name OUT=$ROOT/variants/$name.so EXTRA_NVFLAGS="$flags" -j8
