"""tc_graph_from_csr from pinned vs pageable host arrays (C4): the call's time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
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
ro_p, nb_p = ro.numpy().copy(), nb.numpy().copy()  # pageable copies
for name, (o, b) in (("pinned", (ro, nb)), ("pageable", (ro_p, nb_p))):
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ge = tc.graph_from_csr(o, b, n, E)
        t1 = time.perf_counter()
        del ge
        print(f"{name} from_csr {1e3 * (t1 - t0):.1f} ms", flush=True)
# per-vertex output (134 MB) into pinned vs pageable host memory
ge = tc.graph_from_csr(ro, nb, n, E)
tot = np.zeros(1, np.uint64)
for name, pv in (("pinned", torch.zeros(n, dtype=torch.int64, pin_memory=True)), ("pageable", np.zeros(n, np.uint64))):
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tc.count_triangles_into(ge, tot, pv, tc.MatchOptions(per_vertex=True), sync=True)
        print(f"{name} count+D2H {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
