#!/bin/bash
# GPU box: gpu tests, then C5 (RMAT s26 ef32) whole and 8-part counts, total-only and per-vertex.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 5 gpurun_out/pytest_gpu.log
for pv in 0 1; do
  timeout 900 python tools/phase_probe.py --scale 26 --param 32 --pv $pv --iters 2 > gpurun_out/phases_c5_pv$pv.log 2>&1
  timeout 900 python tools/phase_probe.py --scale 26 --param 32 --pv $pv --iters 2 --parts 8 > gpurun_out/phases_c5_p8_pv$pv.log 2>&1
  echo "== C5 pv=$pv"; grep -v occupancy gpurun_out/phases_c5_pv$pv.log | tail -n 9; tail -n 1 gpurun_out/phases_c5_p8_pv$pv.log
done
