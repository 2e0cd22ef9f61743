import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_02127_b200 as tc
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 12
pv = int(sys.argv[2]) if len(sys.argv) > 2 else 1
pairs = tc.generate(tc.GEN_RMAT, scale, 16)
g = tc.build_graph_from_pairs(pairs, 1 << scale)
print(tc.count_triangles(g, tc.MatchOptions(per_vertex=bool(pv))).count)
