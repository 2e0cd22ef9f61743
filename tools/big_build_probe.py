"""Reproducer for large edge-list builds: RMAT scale/ef on the device, build, count (CUDA_LAUNCH_BLOCKING=1
localises a fault to its launch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_02127_b200 as tc
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 34
m = tc.gen_num_edges(tc.GEN_RMAT, scale, ef)
d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
tc.generate(tc.GEN_RMAT, scale, ef, out=d)
torch.cuda.synchronize()
print("generated", m, flush=True)
rep = tc.BuildReport()
g = tc.build_graph_from_pairs(d, 1 << scale, rep, m=m)
del d
torch.cuda.synchronize()
print("built E", g.num_edges(), rep.self_loops_removed, rep.duplicate_entries_removed, flush=True)
print("T", tc.count_triangles(g).count, flush=True)
