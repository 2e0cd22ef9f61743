import sys, os, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import paper_1909_02127_b200 as tc
pairs = tc.generate(tc.GEN_RMAT, 16, 16)
n = 1 << 16
g = tc.build_graph_from_pairs(pairs, n)
for bins in ("1", "2"):
    os.environ["TCB_DEBUG_BINS"] = bins
    full = tc.count_triangles(g, tc.MatchOptions(per_vertex=False)).count
    for P in (2, 3):
        parts = [tc.count_triangles(g, tc.MatchOptions(per_vertex=False, part_index=p, part_count=P)).count for p in range(P)]
        print("bins", bins, "full", full, "P", P, parts, sum(parts) - full)
