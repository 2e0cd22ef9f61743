#!/bin/bash
# GPU box, one pass for the round's evidence: ncu --set full of the per-count
# kernels (traffic stamped with this build -> profiles/), the default bench
# line (C4), its ncu launch list, the other configs, the reference arm.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_join|k_pv_rows|k_plan" -c 12 -f \
   -o gpurun_out/prof_C4 python tools/prof_count.py --iters 1 --pv 1 > gpurun_out/prof_c4.log 2>&1
python tools/ncu_traffic.py gpurun_out/prof_C4.ncu-rep C4 > gpurun_out/traffic.log 2>&1
cp gpurun_out/ncu_traffic_C4.json profiles/ncu_traffic_C4.json
for k in k_join_cta k_join_dense k_pv_rows; do
  python tools/ncu_summary.py gpurun_out/prof_C4.ncu-rep $k 30 > gpurun_out/sum_$k.txt 2>&1
  python tools/ncu_lines.py gpurun_out/prof_C4.ncu-rep $k 40 > gpurun_out/lines_$k.txt 2>&1
done
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
   python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
for c in C1 C2 C3; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_join_warp" -c 2 -f \
   -o gpurun_out/prof_C2 python tools/prof_count.py --kind er --scale 20 --param 32 --iters 1 --pv 0 > gpurun_out/prof_c2.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_C2.ncu-rep k_join_warp 30 > gpurun_out/sum_k_join_warp_c2.txt 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
for f in gpurun_out/bench_c4.log gpurun_out/bench_C1.log gpurun_out/bench_C2.log gpurun_out/bench_C3.log gpurun_out/bench_ref.log; do echo "== $f"; tail -c 1500 $f; echo; done
timeout 300 python tools/build_probe.py 24 > gpurun_out/build_probe.log 2>&1
timeout 300 python tools/e2e_probe.py 24 > gpurun_out/e2e_probe.log 2>&1
