"""Profiling driver: build a config on the GPU and run N counts (for ncu)."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_02127_b200 as tc
ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="rmat"); ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--param", type=int, default=16); ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--pv", type=int, default=1)
ap.add_argument("--parts", type=int, default=1); ap.add_argument("--part", type=int, default=0)
a = ap.parse_args()
k = {"rmat": tc.GEN_RMAT, "kron": tc.GEN_KRON, "er": tc.GEN_ER}[a.kind]
m = tc.gen_num_edges(k, a.scale, a.param)
d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
tc.generate(k, a.scale, a.param, out=d)
g = tc.build_graph_from_pairs(d, 1 << a.scale, m=m)
del d
for i in range(a.iters):
    r = tc.count_triangles(g, tc.MatchOptions(per_vertex=bool(a.pv), part_index=a.part, part_count=a.parts))
    print(r.count, {k: round(v, 3) if isinstance(v, float) else v for k, v in r.stats.items()})
