#!/bin/bash
# GPU box: bench lines, launch list and a full ncu capture of the join (outputs -> gpurun_out/)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python bench.py --cpu-budget-s 8 > gpurun_out/bench_c4.log 2>&1
for c in C1 C2 C3; do timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 > gpurun_out/bench_$c.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
   python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_join_cta|k_pv_rows|k_fr_scatter|k_join_warp" -c 5 -f \
   -o gpurun_out/prof_c4 python tools/prof_count.py --iters 1 --pv 1 > gpurun_out/prof_c4.log 2>&1
tail -n 2 gpurun_out/*.log
