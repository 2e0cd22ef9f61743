#!/bin/bash
# GPU box: A/B of library variants (variants/*.so) on C4 phases, then the gpu tests on the main build.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
bash tools/ab_phase.sh 1 main ${VARIANTS} > gpurun_out/ab.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 60 gpurun_out/ab.log; tail -n 15 gpurun_out/pytest_gpu.log
