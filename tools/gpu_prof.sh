#!/bin/bash
# GPU box: tests, C4 phases, bench line, ncu full capture of the per-count kernels + traffic stamp.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
T0=$(date +%s)
timeout 1500 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? t=$(( $(date +%s)-T0 ))" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/phase_probe.py --iters 2 > gpurun_out/phases_c4.log 2>&1
timeout 300 python tools/phase_probe.py --iters 1 --parts 8 > gpurun_out/phases_c4_p8.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$? t=$(( $(date +%s)-T0 ))" >> gpurun_out/bench.log
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_join_cta|k_pv_rows|k_join_warp|k_join_small|k_plan" -c 12 -f \
   -o gpurun_out/prof_C4 python tools/prof_count.py --iters 1 --pv 1 > gpurun_out/prof_c4.log 2>&1
python tools/ncu_traffic.py gpurun_out/prof_C4.ncu-rep C4 > gpurun_out/traffic.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_C4.ncu-rep k_join_cta 40 > gpurun_out/join_cta_summary.txt 2>&1
fi
for f in gpurun_out/pytest_gpu.log gpurun_out/phases_c4.log gpurun_out/phases_c4_p8.log gpurun_out/bench.log gpurun_out/traffic.log; do echo "== $f"; tail -n 8 $f; done
