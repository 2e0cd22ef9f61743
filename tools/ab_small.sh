cd $GRAFT_REPO_ROOT
for v in main s32 s64 main s32 s64; do
  lib=variants/$v.so; [ "$v" = "main" ] && lib=paper_1909_02127_b200/libtcb200.so
  echo "== $v C4 pv1"; TCB200_LIB=$PWD/$lib python tools/phase_probe.py --pv 1 --iters 3 2>&1 | grep -E "join_small" | tail -1
  echo "== $v C3 pv0"; TCB200_LIB=$PWD/$lib python tools/phase_probe.py --kind kron --scale 22 --pv 0 --iters 3 2>&1 | grep -E "join_small|total_ms" | tail -2
done
