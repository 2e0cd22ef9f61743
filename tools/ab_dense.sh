#!/bin/bash
# On the GPU box: dense-core parity tests on each variant, then C4 per-vertex phases of main vs the variants.
#   tools/ab_dense.sh var1 var2 ...     (variants/<name>.so from tools/variants.sh)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in "$@"; do
  TCB200_LIB=$PWD/variants/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "dense or stress or golden" > gpurun_out/ab_dense_pytest_$v.log 2>&1
  echo "$v pytest rc=$?"; tail -n 1 gpurun_out/ab_dense_pytest_$v.log
done
bash tools/ab_phase.sh 1 main "$@" main "$@" > gpurun_out/ab_dense_phase.log 2>&1
grep -E "==|dense|total" gpurun_out/ab_dense_phase.log
