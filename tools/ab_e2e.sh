#!/bin/bash
# On the GPU box: e2e phases (from_csr build marks) for library variants.
for v in "$@"; do
  lib=variants/$v.so; [ "$v" = "main" ] && lib=paper_1909_02127_b200/libtcb200.so
  echo "== $v"; TCB200_LIB=$PWD/$lib python tools/e2e_probe.py 24 2>&1 | sed -n "/e2e iter 2/,\$p" | grep -E "fin_|csr_|^e2e"
done
