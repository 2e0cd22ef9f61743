import sys, os, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import paper_1909_02127_b200 as tc
from oracle_ctypes import Oracle
o = Oracle()
pairs = tc.generate(tc.GEN_RMAT, 16, 16)
n = 1 << 16
off, nb, E, _, _ = o.build_graph(pairs, n)
T, pv = o.count(off, nb, per_vertex=True)
g = tc.build_graph_from_pairs(pairs, n)
for i in range(5):
    r = tc.count_triangles(g, tc.MatchOptions(per_vertex=True))
    print('p1', r.count, r.count == T, np.array_equal(r.per_vertex, pv))
for P in (2, 3):
    tot = 0; acc = np.zeros(n, np.uint64)
    for p in range(P):
        r = tc.count_triangles(g, tc.MatchOptions(per_vertex=True, part_index=p, part_count=P))
        print(' part', p, P, r.count, r.stats['segments'])
        tot += r.count; acc += r.per_vertex
    bad = np.nonzero(acc != pv)[0]
    print('P', P, tot, T - tot, 'bad vertices', bad.size, bad[:10], (pv[bad] - acc[bad])[:10] if bad.size else '')
    deg = np.diff(off)
    print('  degs of bad', deg[bad[:10]])
