"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck):
every build route, every join bin (incl. the hash/global-table modes), per-vertex,
multi-part, listings, MatrixMarket and TRIMCSR1 ingest."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np  # noqa: E402

import paper_1909_02127_b200 as tc  # noqa: E402
from oracle_ctypes import Oracle  # noqa: E402

o = Oracle()
pairs = o.gen_rmat(11, 16)
n = 1 << 11
off, nb, E, _, _ = o.build_graph(pairs, n)
T, pv = o.count(off, nb, per_vertex=True)
g = tc.build_graph_from_pairs(pairs, n)
for P in (1, 3):
    tot, acc = 0, np.zeros(n, np.uint64)
    for p in range(P):
        r = tc.count_triangles(g, tc.MatchOptions(per_vertex=True, part_index=p, part_count=P))
        tot += r.count
        acc += r.per_vertex
    assert tot == T and np.array_equal(acc, pv)
g2 = tc.graph_from_csr(off, nb)
assert tc.count_triangles(g2).count == T
rows = tc.list_triangles(g2)
assert rows.shape[0] == T
k = 120
iu, ju = np.triu_indices(k, 1)
kp = np.stack([iu, ju], 1).astype(np.uint32).reshape(-1)
gk = tc.build_graph_from_pairs(kp, k)
assert tc.count_triangles(gk, tc.MatchOptions(per_vertex=True)).count == k * (k - 1) * (k - 2) // 6
text = b"%%MatrixMarket matrix coordinate pattern general\n4 4 3\n1 2\n2 3\n3 1\n"
assert tc.count_triangles(tc.load_matrix_market(text)).count == 1
img = tc.csr_cache_bytes(g)
import ctypes as C  # noqa: E402
h = C.c_void_p()
tc._check(tc._lib.tc_csr_cache_to_graph(img.tobytes(), img.size, 0, C.byref(h)))
assert tc.count_triangles(tc.Graph(h.value, 0)).count == T
# the CSR route streamed in small pieces (rows across piece boundaries) with
# rank-space rows in the lane / warp / <=256 / <=1024 sort classes, and the
# streamed listings
os.environ["TCB_FEED_CHUNK"] = "3000"
k2 = 300
iu, ju = np.triu_indices(k2, 1)
cp = np.concatenate([np.stack([iu, ju], 1).astype(np.uint32).reshape(-1), (pairs + k2).astype(np.uint32)])
off3, nb3, E3, _, _ = o.build_graph(cp, n + k2)
T3 = o.count(off3, nb3)
g3 = tc.graph_from_csr(off3, nb3)
assert tc.count_triangles(g3).count == T3
del os.environ["TCB_FEED_CHUNK"]
assert sum(c.shape[0] for c in tc.iter_listings(g2, max_rows=500)) == T
print("sanitize cases ok", T)
