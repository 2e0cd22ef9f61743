import os, sys
os.environ["TCB_PHASES"] = "1"
sys.path.insert(0, "/root/repo")
import torch
import paper_1909_02127_b200 as tc
scale, ef = 26, 32
m = tc.gen_num_edges(tc.GEN_RMAT, scale, ef); n = 1 << scale
d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
tc.generate(tc.GEN_RMAT, scale, ef, out=d)
g = tc.build_graph_from_pairs(d, n, m=m); del d; torch.cuda.empty_cache()
tot = torch.zeros(1, dtype=torch.int64, device="cuda")
for it in range(2):
    print("--- part 7", file=sys.stderr, flush=True)
    st = tc.count_triangles_into(g, tot, None, tc.MatchOptions(part_index=7, part_count=8), stats=True)
    print(st["total_ms"], st["frontier_ms"], flush=True)
