"""C4 per-vertex counts of the library in TCB200_LIB against the golden FNV (A/B correctness)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch
import paper_1909_02127_b200 as tc
from oracle_ctypes import Oracle
name = sys.argv[1] if len(sys.argv) > 1 else "C4_rmat_s24_ef16"
c = json.load(open(os.path.join(ROOT, "tests", "golden", "synthetic.json")))[name]
k = tc.GEN_ER if c["kind"] == "er" else (tc.GEN_KRON if c["permute"] else tc.GEN_RMAT)
m = tc.gen_num_edges(k, c["scale"], c["edgefactor"])
d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
tc.generate(k, c["scale"], c["edgefactor"], out=d)
g = tc.build_graph_from_pairs(d, c["n"], m=m)
del d
parts = int(os.environ.get("PARTS", "1"))
tot, pv = 0, np.zeros(c["n"], np.uint64)
for p in range(parts):
    r = tc.count_triangles(g, tc.MatchOptions(per_vertex=True, part_index=p, part_count=parts))
    tot += r.count
    pv += r.per_vertex
ok = tot == c["T"] and Oracle().fnv(pv) == c["pv_fnv"]
print(f"pv_check {name} parts={parts}: T={tot} fnv={Oracle().fnv(pv)} {'OK' if ok else 'MISMATCH'}")
