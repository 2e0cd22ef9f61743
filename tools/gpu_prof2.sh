#!/bin/bash
# GPU box: C4 phases + one ncu --set full capture of the per-count kernels (KREGEX).
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python tools/phase_probe.py --iters 2 > gpurun_out/phases_c4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${KREGEX:-k_join}" -c ${NCU_C:-8} -f \
   -o gpurun_out/prof_C4 python tools/prof_count.py --iters 1 --pv ${PV:-1} > gpurun_out/prof_c4.log 2>&1
for k in ${KLIST:-k_join_dense k_join_cta}; do
  python tools/ncu_summary.py gpurun_out/prof_C4.ncu-rep $k 30 > gpurun_out/sum_$k.txt 2>&1
  python tools/ncu_lines.py gpurun_out/prof_C4.ncu-rep $k 30 > gpurun_out/lines_$k.txt 2>&1
done
python tools/ncu_traffic.py gpurun_out/prof_C4.ncu-rep C4 > gpurun_out/traffic.log 2>&1
tail -n 12 gpurun_out/phases_c4.log; for k in ${KLIST:-k_join_dense k_join_cta}; do echo "== $k"; head -32 gpurun_out/sum_$k.txt; head -25 gpurun_out/lines_$k.txt; done
