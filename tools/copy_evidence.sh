#!/bin/bash
# Here (not on the box): copy the outputs of tools/gpu_bench.sh from gpurun_out/ into profiles/ and stamp the
# traffic file with the current commit.
set -e
cd $(dirname $0)/..
G=gpurun_out; P=profiles
for c in c4 C1 C2 C3; do grep '^{' $G/bench_$c.log | tail -1 > $P/r02_bench_$c.json; done
grep '^{' $G/bench_ref.log | tail -1 > $P/r02_bench_ref.json
cp $G/launches_c4.csv $P/r02_launches_c4.csv
python tools/kernel_times.py $P/r02_launches_c4.csv > $P/r02_launches_c4_summary.txt 2>&1
cp $G/sum_k_join_cta.txt $P/r02_ncu_join_cta_c4.txt; cp $G/lines_k_join_cta.txt $P/r02_ncu_join_cta_c4_lines.txt
cp $G/sum_k_join_dense.txt $P/r02_ncu_join_dense_c4.txt; cp $G/lines_k_join_dense.txt $P/r02_ncu_join_dense_c4_lines.txt
cp $G/sum_k_pv_rows.txt $P/r02_ncu_pv_rows_c4.txt; cp $G/sum_k_join_warp_c2.txt $P/r02_ncu_join_warp_c2.txt
cp $G/build_probe.log $P/r02_build_probe_c4.log; cp $G/e2e_probe.log $P/r02_e2e_probe_c4.log
[ -f $G/pytest_gpu_final.log ] && cp $G/pytest_gpu_final.log $P/r02_pytest_gpu_final.log
[ -f $G/phases_c4_p8.log ] && cp $G/phases_c4_p8.log $P/r02_phases_c4_p8_final.log
python - <<PY
import json, subprocess
d = json.load(open("$G/ncu_traffic_C4.json"))
d["git_head"] = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True).stdout.strip()
json.dump(d, open("$P/ncu_traffic_C4.json", "w"), indent=1)
import sys; sys.path.insert(0, ".")
import bench
print("traffic stamp matches sources:", bench.build_inputs_sha256(bench.ROOT) == d["src_sha256"])
for c in ["c4", "C1", "C2", "C3"]:
    b = json.loads(open("$P/r02_bench_%s.json" % c).read()); r = b.get("roofline", {})
    print(c, round(b["value"], 3), b["unit"], "ms", round(b["ms_per_step"], 4), "e2e", round(b["e2e"]["value"], 3),
          "pageable", b["e2e"].get("pageable", {}).get("value"), "frac", r.get("frac"), "traffic", r.get("traffic"),
          r.get("kernels_ms"), b["clocks"])
PY
