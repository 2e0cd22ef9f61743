#!/bin/bash
# On the GPU box: dense-core parity tests on the main build, then C4 phases of main vs the given variants.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "dense or stress or golden" > gpurun_out/ab_dense_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_dense_pytest.log
for pv in 1 0; do bash tools/ab_phase.sh $pv main "$@" main "$@"; done > gpurun_out/ab_dense_phase.log 2>&1
tail -n 2 gpurun_out/ab_dense_pytest.log; grep -E "==|dense|total" gpurun_out/ab_dense_phase.log
