"""C5 (RMAT scale-26 edgefactor-32, ~2.1e9 edges) on one B200: build, whole-graph
count, and the 8-part split run part by part (each part = one rank's work of
an 8-GPU run; max over parts ~ the 8-GPU step without the allreduce)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_02127_b200 as tc  # noqa: E402

scale, ef = 26, 32
pv_on = int(sys.argv[1]) if len(sys.argv) > 1 else 0
m = tc.gen_num_edges(tc.GEN_RMAT, scale, ef)
n = 1 << scale
d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
tc.generate(tc.GEN_RMAT, scale, ef, out=d)
rep = tc.BuildReport()
t0 = time.perf_counter()
g = tc.build_graph_from_pairs(d, n, rep, m=m)
torch.cuda.synchronize()
print(f"build {time.perf_counter() - t0:.2f} s (device {g.build_ms:.0f} ms) E={g.num_edges()} "
      f"loops={rep.self_loops_removed} dups={rep.duplicate_entries_removed} max_d+={g.max_out_degree}", flush=True)
del d
torch.cuda.empty_cache()
E = g.num_edges()
tot = torch.zeros(1, dtype=torch.int64, device="cuda")
pv = torch.zeros(n, dtype=torch.int64, device="cuda") if pv_on else None
out = {"E": E, "per_vertex": bool(pv_on)}
for it in range(2):
    st = tc.count_triangles_into(g, tot, pv, tc.MatchOptions(per_vertex=bool(pv_on)), stats=True)
    out["whole"] = {"T": int(tot.item()), "ms": st["total_ms"], "frontier_ms": st["frontier_ms"],
                    "join_ms": st["join_ms"], "gteps": E / st["total_ms"] / 1e6}
    print("whole", out["whole"], flush=True)
parts = []
for p in range(8):
    st = tc.count_triangles_into(g, tot, pv, tc.MatchOptions(per_vertex=bool(pv_on), part_index=p, part_count=8),
                                 stats=True)
    parts.append({"T": int(tot.item()), "ms": st["total_ms"], "frontier_ms": st["frontier_ms"],
                  "join_ms": st["join_ms"], "J": st["wedges"], "items": st["items"], "segments": st["segments"]})
    print("part", p, parts[-1], flush=True)
out["parts8"] = parts
out["parts8_sum_T"] = sum(p["T"] for p in parts)
out["parts8_max_ms"] = max(p["ms"] for p in parts)
out["parts8_gteps_at_max"] = E / out["parts8_max_ms"] / 1e6
print(json.dumps(out), flush=True)
