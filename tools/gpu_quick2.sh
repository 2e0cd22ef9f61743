#!/bin/bash
# GPU box: smoke, gpu tests, C4 phases (whole, 8 parts), C3.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/phase_probe.py --iters 2 > gpurun_out/phases_c4.log 2>&1
timeout 300 python tools/phase_probe.py --iters 2 --parts 8 > gpurun_out/phases_c4_p8.log 2>&1
for f in gpurun_out/smoke.log gpurun_out/pytest_gpu.log; do echo "== $f"; tail -n 6 $f; done
for f in gpurun_out/phases_c4.log gpurun_out/phases_c4_p8.log; do echo "== $f"; grep -v occupancy $f | tail -n 12; done
