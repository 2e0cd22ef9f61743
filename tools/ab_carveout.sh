#!/bin/bash
# GPU box: join time vs shared-memory carveout: tools/ab_carveout.sh variant "c1 c2 ..."
v=$1; lib=variants/$v.so; [ "$v" = "main" ] && lib=paper_1909_02127_b200/libtcb200.so
for c in $2; do
  echo "== $v carveout=$c"
  if [ "$c" = "def" ]; then TCB200_LIB=$PWD/$lib python tools/phase_probe.py --pv ${PV:-1} --iters 2 2>&1 | grep -E "occupancy|join_cta|total" | tail -4
  else TCB_CARVEOUT=$c TCB200_LIB=$PWD/$lib python tools/phase_probe.py --pv ${PV:-1} --iters 2 2>&1 | grep -E "occupancy|join_cta|total" | tail -4; fi
done
