"""Per-phase device times of tc_count on one config (TCB_PHASES=1 prints them)."""
import argparse
import os
import sys

os.environ.setdefault("TCB_PHASES", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_02127_b200 as tc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="rmat")
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--param", type=int, default=16)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--pv", type=int, default=1)
ap.add_argument("--parts", type=int, default=1)
ap.add_argument("--work", type=int, default=0, help="1: work counters (TCB_PHASES prints the plan sums)")
a = ap.parse_args()
k = {"rmat": tc.GEN_RMAT, "kron": tc.GEN_KRON, "er": tc.GEN_ER}[a.kind]
m = tc.gen_num_edges(k, a.scale, a.param)
d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
tc.generate(k, a.scale, a.param, out=d)
g = tc.build_graph_from_pairs(d, 1 << a.scale, m=m)
del d
torch.cuda.empty_cache()
print(f"graph: |E|={g.num_edges()} build_ms={g.build_ms:.1f} core_ranks={g.core_ranks} dense_rows={g.dense_rows}",
      flush=True)
n = 1 << a.scale
tot = torch.zeros(1, dtype=torch.int64, device="cuda")
pv = torch.zeros(n, dtype=torch.int64, device="cuda") if a.pv else None
for i in range(a.iters):
    print(f"--- iter {i}", file=sys.stderr, flush=True)
    T, ms, per = 0, {}, []
    for p in range(a.parts):
        st = tc.count_triangles_into(g, tot, pv, tc.MatchOptions(per_vertex=bool(a.pv), part_index=p,
                                                                 part_count=a.parts), stats=True,
                                   work_counters=bool(a.work))
        T += int(tot.item())
        per.append(round(st["total_ms"], 2))
        if a.parts > 1 and i == a.iters - 1:
            print(f"  part {p}: " + " ".join(f"{k[:-3]}={st[k]:.2f}" for k in
                                          ("frontier_ms", "warp_ms", "small_ms", "cta_ms", "dense_ms", "rows_ms")),
                  flush=True)
        for k, v in st.items():
            if k.endswith("_ms"):
                ms[k] = ms.get(k, 0) + v
    print(T, {k: round(v, 3) for k, v in ms.items()}, flush=True)
    if a.parts > 1:
        print(f"parts={a.parts} max={max(per)} sum={round(sum(per), 2)} per={per}", flush=True)
