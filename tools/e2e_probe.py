"""Phase times of the drop-in e2e path (host CSR -> tc_graph_from_csr -> tc_count -> host)."""
import os
import sys
import time

os.environ.setdefault("TCB_PHASES", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_02127_b200 as tc  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
m = tc.gen_num_edges(tc.GEN_RMAT, scale, 16)
d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
tc.generate(tc.GEN_RMAT, scale, 16, out=d)
n = 1 << scale
g = tc.build_graph_from_pairs(d, n, m=m)
del d
E = g.num_edges()
ro = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
nb = torch.empty(2 * E, dtype=torch.int32, pin_memory=True)
g.export_csr(ro, nb)
del g
tot = torch.zeros(1, dtype=torch.int64, pin_memory=True)
pv = torch.zeros(n, dtype=torch.int64, pin_memory=True)
for i in range(3):
    print(f"--- e2e iter {i}", file=sys.stderr, flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ge = tc.graph_from_csr(ro, nb, n, E)
    t1 = time.perf_counter()
    tc.count_triangles_into(ge, tot, pv, tc.MatchOptions(per_vertex=True), sync=True)
    t2 = time.perf_counter()
    del ge
    print(f"e2e {1e3*(t2-t0):.1f} ms: from_csr {1e3*(t1-t0):.1f} count {1e3*(t2-t1):.1f} T={int(tot[0])}", flush=True)
# raw link bandwidth for reference
dst = torch.empty_like(nb, device="cuda")
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dst.copy_(nb, non_blocking=True)
    torch.cuda.synchronize()
    print(f"raw H2D {nb.numel()*4/1e9:.2f} GB: {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
