"""Whole-count CUDA graph replay vs direct launches (per config)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_02127_b200 as tc  # noqa: E402

for kind, scale, param, pv in (("rmat", 16, 16, False), ("er", 20, 32, False), ("kron", 22, 16, False),
                               ("rmat", 24, 16, True)):
    k = {"rmat": tc.GEN_RMAT, "kron": tc.GEN_KRON, "er": tc.GEN_ER}[kind]
    m = tc.gen_num_edges(k, scale, param)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    tc.generate(k, scale, param, out=d)
    g = tc.build_graph_from_pairs(d, 1 << scale, m=m)
    del d
    g.set_stream(st.cuda_stream)
    n = 1 << scale
    with torch.cuda.stream(st):
        tot = torch.zeros(1, dtype=torch.int64, device="cuda")
        pvb = torch.zeros(n, dtype=torch.int64, device="cuda") if pv else None
    torch.cuda.synchronize()
    opts = tc.MatchOptions(per_vertex=pv)
    for _ in range(3):
        tc.count_triangles_into(g, tot, pvb, opts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 20
    e0.record(st)
    for _ in range(K):
        tc.count_triangles_into(g, tot, pvb, opts)
    e1.record(st)
    torch.cuda.synchronize()
    direct = e0.elapsed_time(e1) / K
    T0 = int(tot.item())
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg, stream=st, capture_error_mode="relaxed"):
        tc.count_triangles_into(g, tot, pvb, opts)
    torch.cuda.synchronize()
    tot.zero_()
    with torch.cuda.stream(st):
        for _ in range(3):
            cg.replay()
    torch.cuda.synchronize()
    e0.record(st)
    with torch.cuda.stream(st):
        for _ in range(K):
            cg.replay()
    e1.record(st)
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / K
    T1 = int(tot.item())
    E = g.num_edges()
    del cg, g
    torch.cuda.synchronize()
    print(f"{kind} s{scale}: T={T0} graphT={T1} direct {direct:.4f} ms graph {graph:.4f} ms "
          f"({E / graph / 1e6:.2f} GTEPS)", flush=True)
