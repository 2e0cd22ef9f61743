"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden
vectors and the oracle, bit-exact (integer work: no tolerance)."""
import os

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _pairs(case):
    return np.array(case.get("pairs", case.get("edges", [])), dtype=np.uint32).reshape(-1)


def _count(tc, g, pv=True):
    r = tc.count_triangles(g, tc.MatchOptions(per_vertex=pv))
    return r


def test_known_answers(tc, cuda_ok):
    for name, c in load_golden("known.json").items():
        if name.startswith("_"):
            continue
        rep = tc.BuildReport()
        g = tc.build_graph(tc.EdgeList(c["n"], _pairs(c)), rep)
        assert g.num_edges() == c["E"], name
        assert (rep.self_loops_removed, rep.duplicate_entries_removed) == (c["loops"], c["dups"]), name
        r = _count(tc, g, pv=not c.get("skip_ref_csr"))
        assert r.count == c["T"], name
        if c.get("skip_ref_csr"):
            continue
        assert r.per_vertex.tolist() == c["per_vertex"], name
        ro, nb = g.export_csr()
        assert ro.tolist() == c["offsets"], name
        assert nb.tolist() == c["nbrs"], name
        assert tc.degrees(g).tolist() == np.diff(np.array(c["offsets"], np.int64)).tolist(), name


def test_high_ids_and_huge_declared_n(tc, cuda_ok):
    c = load_golden("known.json")["K3_high_ids"]
    g = tc.build_graph(tc.EdgeList(c["n"], _pairs(c)))
    assert g.num_vertices() == 0xFFFFFFFF and g.num_edges() == 3
    assert tc.count_triangles(g).count == 1


def test_errors(tc, cuda_ok):
    with pytest.raises(tc.InvalidArgument):
        tc.build_graph(tc.EdgeList(3, np.array([[0, 5]], np.uint32)))
    with pytest.raises(tc.InvalidArgument):
        tc.build_graph(tc.EdgeList(0, np.array([[0, 0]], np.uint32)))
    g = tc.build_graph(tc.EdgeList(3, np.array([[0, 1], [1, 2], [0, 2]], np.uint32)))
    with pytest.raises(tc.InvalidArgument):
        tc.count_triangles(g, tc.MatchOptions(lookahead=3))
    r = tc.count_triangles(g, tc.MatchOptions(keep_listings=True))
    assert r.count == 1 and r.listings.tolist() == [[0, 1, 2]]
    with pytest.raises(IndexError):
        g.has_edge(0, 3)
    assert g.has_edge(0, 2) and not g.has_edge(0, 0)
    for la in (0, 1, 2):
        assert tc.count_triangles(g, tc.MatchOptions(lookahead=la)).count == 1


def test_gnp_golden(tc, cuda_ok):
    for i, c in enumerate(load_golden("gnp.json")):
        rep = tc.BuildReport()
        g = tc.build_graph(tc.EdgeList(c["n"], _pairs(c)), rep)
        assert (g.num_edges(), rep.self_loops_removed, rep.duplicate_entries_removed) == \
            (c["E"], c["loops"], c["dups"]), i
        r = _count(tc, g)
        assert r.count == c["T"], i
        assert r.per_vertex.tolist() == c["per_vertex"], i


def test_gnp_500_vs_oracle(tc, oracle, cuda_ok):
    rng = np.random.default_rng(7)
    for i in range(510):
        n = int(rng.integers(20, 201))
        p = (0.02, 0.1, 0.3)[i % 3]
        iu, ju = np.triu_indices(n, 1)
        keep = rng.random(iu.size) < p
        pairs = np.stack([iu[keep], ju[keep]], 1).astype(np.uint32).reshape(-1)
        off, nb, E, _, _ = oracle.build_graph(pairs, n)
        T, pv = oracle.count(off, nb, per_vertex=True)
        g = tc.build_graph_from_pairs(pairs, n)
        r = _count(tc, g)
        assert r.count == T and np.array_equal(r.per_vertex, pv), i
        # the Graph-ctor route (count_triangles(const Graph&))
        g2 = tc.graph_from_csr(off, nb)
        assert tc.count_triangles(g2).count == T, i


def test_build_graph_csr_parity_random(tc, oracle, cuda_ok):
    rng = np.random.default_rng(3)
    for i in range(60):
        n = int(rng.integers(1, 3000))
        m = int(rng.integers(0, 20 * n))
        pairs = rng.integers(0, n, 2 * m).astype(np.uint32)
        if m and i % 3 == 0:  # heavy duplication + loops
            pairs[: m // 2] = pairs[0]
        off, nb, E, lo, du = oracle.build_graph(pairs, n)
        rep = tc.BuildReport()
        g = tc.build_graph_from_pairs(pairs, n, rep)
        assert (g.num_edges(), rep.self_loops_removed, rep.duplicate_entries_removed) == (E, lo, du)
        ro, nbr = g.export_csr()
        assert np.array_equal(ro, off) and np.array_equal(nbr, nb), i


def test_export_csr_chunked(tc, oracle, cuda_ok):
    """tc_graph_export_csr by source-id ranges (the path graphs with >= 2^31
    directed entries take; TCB_EXPORT_CHUNK shrinks the range here)."""
    rng = np.random.default_rng(13)
    old = os.environ.get("TCB_EXPORT_CHUNK")
    try:
        for i, chunk in enumerate(("1000", "4096", "1")):
            os.environ["TCB_EXPORT_CHUNK"] = chunk
            n = int(rng.integers(50, 3000))
            m = int(rng.integers(n, 12 * n))
            pairs = rng.integers(0, n, 2 * m).astype(np.uint32)
            off, nb, E, _, _ = oracle.build_graph(pairs, n)
            g = tc.build_graph_from_pairs(pairs, n)
            if chunk == "1" and int(np.diff(off).max()) > 1:
                with pytest.raises(IndexError):
                    g.export_csr()
                continue
            ro, nbr = g.export_csr()
            assert np.array_equal(ro, off) and np.array_equal(nbr, nb), i
    finally:
        if old is None:
            os.environ.pop("TCB_EXPORT_CHUNK", None)
        else:
            os.environ["TCB_EXPORT_CHUNK"] = old


def _stress_graphs():
    # hubs / cliques: force every bin, large tables and the global-table path
    out = {}
    n = 4000
    star = np.array([[0, i] for i in range(1, n)], np.uint32)
    ring = np.array([[i, i + 1] for i in range(1, n - 1)], np.uint32)
    out["wheel"] = (n, np.concatenate([star, ring]))
    k = 300
    iu, ju = np.triu_indices(k, 1)
    out["K300"] = (k, np.stack([iu, ju], 1).astype(np.uint32))
    rng = np.random.default_rng(5)
    # dense core (large d+) + sparse fringe attached to it
    core = 1200
    iu, ju = np.triu_indices(core, 1)
    keep = rng.random(iu.size) < 0.5
    dense = np.stack([iu[keep], ju[keep]], 1)
    fringe = np.stack([rng.integers(core, 60000, 200000), rng.integers(0, core, 200000)], 1)
    out["core_fringe"] = (60000, np.concatenate([dense, fringe]).astype(np.uint32))
    return out


# membership / counter paths: default windows; tiny windows (most members in
# the hash, most per-vertex hits as global atomics); hash forced to the global
# slab
MODES = {
    "default": {},
    "hash": {"TCB_HOT_BITS": "64", "TCB_TOP_COUNTERS": "32"},
    "global_table": {"TCB_HOT_BITS": "64", "TCB_TOP_COUNTERS": "16", "TCB_SMEM_SLOTS": "32"},
    # dense core (RowGeo): a small core with a low threshold makes most rows
    # dense; no core at all (every row sparse)
    "dense_small": {"TCB_CORE_BITS": "96", "TCB_CORE_MIN": "1"},
    "dense_hash": {"TCB_HOT_BITS": "256", "TCB_CORE_BITS": "224", "TCB_CORE_MIN": "2", "TCB_TOP_COUNTERS": "32"},
    "no_core": {"TCB_CORE_BITS": "0"},
}


@pytest.fixture
def mode_env(request):
    env = MODES[request.param]
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    yield request.param
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


@pytest.mark.parametrize("mode_env", list(MODES), indirect=True)
@pytest.mark.parametrize("name", ["wheel", "K300", "core_fringe"])
def test_stress_bins(tc, oracle, cuda_ok, name, mode_env):
    n, e = _stress_graphs()[name]
    pairs = e.reshape(-1)
    off, nb, E, _, _ = oracle.build_graph(pairs, n)
    T, pv = oracle.count(off, nb, per_vertex=True)
    g = tc.build_graph_from_pairs(pairs, n)
    r = _count(tc, g)
    assert r.count == T and np.array_equal(r.per_vertex, pv)
    assert tc.count_triangles(g, tc.MatchOptions(per_vertex=False)).count == T


@pytest.mark.parametrize("mode_env", ["default", "global_table", "no_core"], indirect=True)
def test_large_clique(tc, cuda_ok, mode_env):
    # K_k: d+ up to k-1 -> 16K-slot tables
    k = 6000
    a = np.repeat(np.arange(k, dtype=np.uint32), np.arange(k - 1, -1, -1))
    b = np.concatenate([np.arange(i + 1, k, dtype=np.uint32) for i in range(k)])
    pairs = np.stack([a, b], 1).reshape(-1)
    g = tc.build_graph_from_pairs(pairs, k)
    T = k * (k - 1) * (k - 2) // 6
    r = _count(tc, g)
    assert r.count == T
    assert np.all(r.per_vertex == (k - 1) * (k - 2) // 2)


@pytest.mark.parametrize("mode_env", ["dense_small", "dense_hash"], indirect=True)
def test_gnp_dense_core(tc, oracle, cuda_ok, mode_env):
    """The dense-core step (word-parallel core intersections, graph.cuh
    RowGeo) against the oracle: every bin, both routes, per-vertex, parts."""
    rng = np.random.default_rng(11)
    for i in range(90):
        n = int(rng.integers(64, 700))
        p = (0.05, 0.2, 0.5)[i % 3]
        iu, ju = np.triu_indices(n, 1)
        keep = rng.random(iu.size) < p
        pairs = np.stack([iu[keep], ju[keep]], 1).astype(np.uint32).reshape(-1)
        off, nb, E, _, _ = oracle.build_graph(pairs, n)
        T, pv = oracle.count(off, nb, per_vertex=True)
        g = tc.build_graph_from_pairs(pairs, n)
        r = _count(tc, g)
        assert r.count == T and np.array_equal(r.per_vertex, pv), i
        assert tc.count_triangles(g, tc.MatchOptions(per_vertex=False)).count == T, i
        g2 = tc.graph_from_csr(off, nb)
        assert tc.count_triangles(g2).count == T, i
        if i % 9 == 0:
            tot, acc = 0, np.zeros(n, np.uint64)
            for q in range(3):
                rq = tc.count_triangles(g, tc.MatchOptions(per_vertex=True, part_index=q, part_count=3))
                tot += rq.count
                acc += rq.per_vertex
            assert tot == T and np.array_equal(acc, pv), i


@pytest.mark.parametrize("parts", [2, 3, 8])
def test_parts_sum_to_total_er(tc, oracle, cuda_ok, parts):
    """Multi-part sums on a uniform-degree graph (ER, every pivot in the warp bin)."""
    c = load_golden("synthetic.json")["C2_er_s20_d32"]
    pairs = tc.generate(tc.GEN_ER, 20, 32)
    g = tc.build_graph_from_pairs(pairs, c["n"])
    assert g.max_out_degree <= 48
    tot = 0
    pv = np.zeros(c["n"], np.uint64)
    for p in range(parts):
        r = tc.count_triangles(g, tc.MatchOptions(per_vertex=True, part_index=p, part_count=parts))
        tot += r.count
        pv += r.per_vertex
    assert tot == c["T"]
    assert oracle.fnv(pv) == c["pv_fnv"]


@pytest.mark.parametrize("parts", [2, 3, 8])
def test_parts_sum_to_total(tc, oracle, cuda_ok, parts):
    c = load_golden("synthetic.json")["C1_rmat_s16_ef16"]
    pairs = tc.generate(tc.GEN_RMAT, 16, 16)
    g = tc.build_graph_from_pairs(pairs, c["n"])
    tot = 0
    pv = np.zeros(c["n"], np.uint64)
    for p in range(parts):
        r = tc.count_triangles(g, tc.MatchOptions(per_vertex=True, part_index=p, part_count=parts))
        tot += r.count
        pv += r.per_vertex
    assert tot == c["T"]
    assert oracle.fnv(pv) == c["pv_fnv"]


@pytest.mark.parametrize("parts", [1, 3, 8])
def test_count_multi_one_gpu(tc, oracle, cuda_ok, parts):
    """tc_count_multi: P parts of the pivot split on device 0 --
    counted back to back, summed, then the NCCL allreduce (a 1-rank
    communicator here) -- against the reference goldens."""
    c = load_golden("synthetic.json")["C1_rmat_s16_ef16"]
    g = tc.build_graph_from_pairs(tc.generate(tc.GEN_RMAT, 16, 16), c["n"])
    mg = tc.MultiGPU([0] * parts)
    r = mg.count_triangles([g] * parts, tc.MatchOptions(per_vertex=True))
    assert r.count == c["T"]
    assert oracle.fnv(r.per_vertex) == c["pv_fnv"]
    r2 = mg.count_triangles([g] * parts)
    assert r2.count == c["T"] and r2.per_vertex is None
    # device outputs
    import torch
    tot = torch.zeros(1, dtype=torch.int64, device="cuda")
    pv = torch.zeros(c["n"], dtype=torch.int64, device="cuda")
    mg.count_triangles([g] * parts, tc.MatchOptions(per_vertex=True), total=tot, per_vertex=pv)
    assert int(tot.item()) == c["T"]
    assert oracle.fnv(pv.cpu().numpy().view(np.uint64)) == c["pv_fnv"]
    mg.close()


def test_comm_allreduce_single_rank(tc, oracle, cuda_ok):
    """tc_comm_init_rank + tc_count_allreduce (one process per GPU) with a
    1-rank group: the count path plus the NCCL allreduce on the count stream."""
    c = load_golden("synthetic.json")["C2_er_s20_d32"]
    g = tc.build_graph_from_pairs(tc.generate(tc.GEN_ER, 20, 32), c["n"])
    comm = tc.Comm(tc.Comm.unique_id(), 1, 0, 0)
    r = comm.count_triangles(g, tc.MatchOptions(per_vertex=True))
    assert r.count == c["T"]
    assert oracle.fnv(r.per_vertex) == c["pv_fnv"]
    assert comm.count_triangles(g).count == c["T"]
    comm.close()


def test_multi_errors(tc, cuda_ok):
    g1 = tc.build_graph_from_pairs(np.array([0, 1, 1, 2, 2, 0], np.uint32), 3)
    g2 = tc.build_graph_from_pairs(np.array([0, 1, 1, 2], np.uint32), 3)
    mg = tc.MultiGPU([0, 0])
    with pytest.raises(tc.InvalidArgument):
        mg.count_triangles([g1, g2])  # not replicas
    with pytest.raises(tc.InvalidArgument):
        mg.count_triangles([g1])      # one graph per part
    with pytest.raises(tc.InvalidArgument):
        tc.Comm(b"x" * 12, 1, 0, 0)
    mg.close()


@pytest.mark.slow
def test_c4_count_multi_8_parts(tc, oracle, cuda_ok):
    syn = load_golden("synthetic.json")
    c = syn["C4_rmat_s24_ef16"]
    import torch
    m = tc.gen_num_edges(tc.GEN_RMAT, 24, 16)
    d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
    tc.generate(tc.GEN_RMAT, 24, 16, out=d)
    g = tc.build_graph_from_pairs(d, c["n"], m=m)
    del d
    mg = tc.MultiGPU([0] * 8)
    r = mg.count_triangles([g] * 8, tc.MatchOptions(per_vertex=True))
    assert r.count == c["T"]
    assert oracle.fnv(r.per_vertex) == c["pv_fnv"]
    mg.close()


def test_partition_bounds_match_host(tc, oracle, cuda_ok):
    import dist_ref
    pairs = tc.generate(tc.GEN_RMAT, 14, 16)
    g = tc.build_graph_from_pairs(pairs, 1 << 14)
    off, nb, E, _, _ = oracle.build_graph(pairs, 1 << 14)
    roff, col, src, order = dist_ref.degree_rank_dag(off, nb)
    cost = dist_ref.pivot_cost(roff, col, src)
    for P in (2, 3, 8):
        assert tc.partition_bounds(g, P).tolist() == \
            dist_ref.partition_bounds(cost, P, dist_ref.isolated(off)).tolist()


SYN = ["C1_rmat_s16_ef16", "C2_er_s20_d32", "rmat_s18_ef16", "kron_s18_ef16", "rmat_s20_ef16"]


@pytest.mark.parametrize("name", SYN)
def test_synthetic_golden(tc, oracle, cuda_ok, name):
    c = load_golden("synthetic.json")[name]
    kind = tc.GEN_ER if c["kind"] == "er" else (tc.GEN_KRON if c["permute"] else tc.GEN_RMAT)
    pairs = tc.generate(kind, c["scale"], c["edgefactor"])
    assert oracle.fnv(pairs) == c["pairs_fnv"]
    rep = tc.BuildReport()
    g = tc.build_graph_from_pairs(pairs, c["n"], rep)
    assert (g.num_edges(), rep.self_loops_removed, rep.duplicate_entries_removed) == (c["E"], c["loops"], c["dups"])
    r = _count(tc, g)
    assert r.count == c["T"]
    assert oracle.fnv(r.per_vertex) == c["pv_fnv"]
    assert int(r.per_vertex.sum()) == 3 * c["T"] == c["pv_sum"]
    ro, nb = g.export_csr()
    assert oracle.fnv(ro) == c["offsets_fnv"] and oracle.fnv(nb) == c["nbrs_fnv"]
    # Graph-ctor route from the exported CSR gives the same answer
    g2 = tc.graph_from_csr(ro, nb)
    assert tc.count_triangles(g2).count == c["T"]


def test_device_resident_inputs(tc, cuda_ok):
    import torch
    c = load_golden("synthetic.json")["C2_er_s20_d32"]
    m = tc.gen_num_edges(tc.GEN_ER, 20, 32)
    d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
    tc.generate(tc.GEN_ER, 20, 32, out=d)
    g = tc.build_graph_from_pairs(d, c["n"], m=m)
    total = torch.zeros(1, dtype=torch.int64, device="cuda")
    pv = torch.zeros(c["n"], dtype=torch.int64, device="cuda")
    tc.count_triangles_into(g, total, pv, tc.MatchOptions(per_vertex=True), sync=True)
    assert int(total.item()) == c["T"]
    assert int(pv.sum().item()) == 3 * c["T"]


def test_csr_cache_roundtrip(tc, tmp_path, cuda_ok):
    c = load_golden("known.json")["two_K4_share_edge"]
    g = tc.build_graph(tc.EdgeList(c["n"], _pairs(c)))
    p = str(tmp_path / "g.trimcsr")
    tc.write_csr_cache(p, g)
    g2 = tc.load_graph(p)
    assert g2.num_edges() == c["E"] and tc.count_triangles(g2).count == c["T"]
    mm = tmp_path / "g.mtx"
    mm.write_text("%%MatrixMarket matrix coordinate pattern general\n6 6 3\n1 2\n2 3\n3 1\n")
    rep = tc.BuildReport()
    g3 = tc.load_graph(str(mm), rep)
    assert tc.count_triangles(g3).count == 1


@pytest.mark.slow
def test_c3_kron_s22(tc, oracle, cuda_ok):
    syn = load_golden("synthetic.json")
    if "C3_kron_s22_ef16" not in syn:
        pytest.skip("C3 golden not generated")
    c = syn["C3_kron_s22_ef16"]
    import torch
    m = tc.gen_num_edges(tc.GEN_KRON, 22, 16)
    d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
    tc.generate(tc.GEN_KRON, 22, 16, out=d)
    rep = tc.BuildReport()
    g = tc.build_graph_from_pairs(d, c["n"], rep, m=m)
    assert (g.num_edges(), rep.self_loops_removed, rep.duplicate_entries_removed) == (c["E"], c["loops"], c["dups"])
    r = _count(tc, g)
    assert r.count == c["T"]
    assert oracle.fnv(r.per_vertex) == c["pv_fnv"]


@pytest.mark.slow
def test_c4_rmat_s24(tc, oracle, cuda_ok):
    syn = load_golden("synthetic.json")
    if "C4_rmat_s24_ef16" not in syn:
        pytest.skip("C4 golden not generated")
    c = syn["C4_rmat_s24_ef16"]
    import torch
    m = tc.gen_num_edges(tc.GEN_RMAT, 24, 16)
    d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
    tc.generate(tc.GEN_RMAT, 24, 16, out=d)
    rep = tc.BuildReport()
    g = tc.build_graph_from_pairs(d, c["n"], rep, m=m)
    del d
    assert (g.num_edges(), rep.self_loops_removed, rep.duplicate_entries_removed) == (c["E"], c["loops"], c["dups"])
    assert g.core_ranks == 2048 and g.dense_rows > 100000  # the dense-core step carries ~45% of the wedges here
    r = _count(tc, g)
    assert r.count == c["T"] == 10282799137
    assert oracle.fnv(r.per_vertex) == c["pv_fnv"]
    assert int(r.per_vertex.sum()) == 3 * c["T"]
    assert tc.count_triangles(g, tc.MatchOptions(per_vertex=False)).count == c["T"]


# ---- the Graph-ctor (CSR) route: per-row orientation, hub chunks, row sorts ----

def _clique_pairs(k, base=0):
    iu, ju = np.triu_indices(k, 1)
    return np.stack([iu + base, ju + base], 1).astype(np.uint32)


@pytest.mark.parametrize("rowsort", ["default", "radix_fallback", "streamed"])
def test_csr_route_paths(tc, oracle, cuda_ok, rowsort):
    """Hub rows longer than one 1024-entry chunk, rank-space rows in every
    sort class (<=16 lane network, 17..32 warp, 33..256, 257..1024, >1024
    CTA), the radix fallback, and the host neighbour array streamed in 4096-
    entry pieces (rows, hub rows included, span piece boundaries); counts,
    per-vertex counts and the exported CSR must match the oracle."""
    old = os.environ.get("TCB_ROWSORT_MAX")
    if rowsort == "radix_fallback":
        os.environ["TCB_ROWSORT_MAX"] = "32"
    if rowsort == "streamed":
        os.environ["TCB_FEED_CHUNK"] = "4096"
    try:
        rng = np.random.default_rng(11)
        parts = [_clique_pairs(1300), _clique_pairs(300, 1300), _clique_pairs(60, 1600), _clique_pairs(24, 1660)]
        n = 9000
        hub = np.stack([np.full(n - 1700, 1690, np.uint32), np.arange(1700, n, dtype=np.uint32)], 1)
        fringe = np.stack([rng.integers(1700, n, 30000), rng.integers(0, 1700, 30000)], 1).astype(np.uint32)
        pairs = np.concatenate(parts + [hub, fringe]).reshape(-1)
        off, nb, E, _, _ = oracle.build_graph(pairs, n)
        T, pv = oracle.count(off, nb, per_vertex=True)
        g = tc.graph_from_csr(off, nb)
        assert g.num_edges() == E and g.max_out_degree >= 1100
        r = _count(tc, g)
        assert r.count == T and np.array_equal(r.per_vertex, pv)
        ro, nbr = g.export_csr()
        assert np.array_equal(ro, off) and np.array_equal(nbr, nb)
        assert np.array_equal(tc.degrees(g), np.diff(off).astype(np.uint32))
    finally:
        os.environ.pop("TCB_FEED_CHUNK", None)
        if old is None:
            os.environ.pop("TCB_ROWSORT_MAX", None)
        else:
            os.environ["TCB_ROWSORT_MAX"] = old


def test_csr_route_errors(tc, cuda_ok):
    """Graph ctor validation (graph.cpp:9-21): inconsistent arrays and ids out
    of range raise std::invalid_argument (InvalidArgument)."""
    off = np.array([0, 2, 4, 6], np.uint64)
    nb = np.array([1, 2, 0, 2, 0, 1], np.uint32)
    assert tc.count_triangles(tc.graph_from_csr(off, nb)).count == 1
    with pytest.raises(tc.InvalidArgument):  # asymmetric: 0->1 without 1->0
        tc.graph_from_csr(np.array([0, 2, 3, 5], np.uint64), np.array([1, 2, 2, 0, 1], np.uint32), 3, 3)
    with pytest.raises(tc.InvalidArgument):  # neighbour id out of range
        tc.graph_from_csr(off, np.array([1, 7, 0, 2, 0, 1], np.uint32))
    with pytest.raises(tc.InvalidArgument):  # decreasing offsets
        tc.graph_from_csr(np.array([0, 4, 2, 6], np.uint64), nb)
    with pytest.raises(tc.InvalidArgument):  # offsets[n] != 2|E|
        tc.graph_from_csr(np.array([0, 2, 4, 5], np.uint64), nb, 3, 3)


# ---- on-disk formats through the device ----

def _csr_image(nv, off, nb):
    return (b"TRIMCSR1" + np.array([1, nv, len(nb) // 2], "<u8").tobytes() + np.asarray(off, "<u8").tobytes()
            + np.asarray(nb, "<u4").tobytes())


def test_csr_cache_corruption(tc, cuda_ok):
    """read_csr_cache invariants (io.cpp:206-218), checked on the device with
    the reference's messages: offsets first, then adjacency."""
    import ctypes as C
    ok = _csr_image(3, [0, 2, 4, 6], [1, 2, 0, 2, 0, 1])
    h = C.c_void_p()
    tc._check(tc._lib.tc_csr_cache_to_graph(ok, len(ok), 0, C.byref(h)))
    tc._lib.tc_graph_destroy(h)
    cases = {
        "corrupt CSR cache offsets": [_csr_image(3, [1, 2, 4, 6], [1, 2, 0, 2, 0, 1]),   # front != 0
                                      _csr_image(3, [0, 4, 2, 6], [1, 2, 0, 2, 0, 1])],  # decreasing
        "corrupt CSR cache adjacency": [_csr_image(3, [0, 2, 4, 6], [2, 1, 0, 2, 0, 1]),  # not ascending
                                        _csr_image(3, [0, 2, 4, 6], [0, 2, 0, 2, 0, 1]),  # self-loop
                                        _csr_image(3, [0, 2, 4, 6], [1, 9, 0, 2, 0, 1]),  # out of range
                                        _csr_image(3, [0, 2, 4, 6], [1, 1, 0, 2, 0, 1])],  # duplicate
    }
    for msg, imgs in cases.items():
        for img in imgs:
            with pytest.raises(tc.ParseError) as ei:
                tc._check(tc._lib.tc_csr_cache_to_graph(img, len(img), 0, C.byref(C.c_void_p())))
            assert msg in str(ei.value) and ei.value.line == 1


def test_csr_cache_emit_roundtrip(tc, oracle, cuda_ok):
    """write_csr_cache from the device graph == the reference's byte layout,
    and reads back to the same graph."""
    pairs = tc.generate(tc.GEN_RMAT, 12, 16)
    off, nb, E, _, _ = oracle.build_graph(pairs, 1 << 12)
    g = tc.build_graph_from_pairs(pairs, 1 << 12)
    img = tc.csr_cache_bytes(g)
    assert img.tobytes() == _csr_image(1 << 12, off, nb)
    import ctypes as C
    h = C.c_void_p()
    tc._check(tc._lib.tc_csr_cache_to_graph(img.tobytes(), img.size, 0, C.byref(h)))
    g2 = tc.Graph(h.value, 0)
    assert g2.num_edges() == E and tc.count_triangles(g2).count == oracle.count(off, nb)


def _mm_text(rng, n, m, *, crlf=False, values=False, comments=True):
    lines = ["%%MatrixMarket matrix coordinate pattern general", "% generated"]
    ij = rng.integers(1, n + 1, (m, 2))
    lines.append(f"{n} {n} {m}")
    for k, (i, j) in enumerate(ij):
        if comments and k % 7 == 3:
            lines.append("% a comment")
        if comments and k % 11 == 5:
            lines.append("   ")
        sep = "\t" if k % 3 == 0 else " " * (1 + k % 2)
        lines.append(f"{i}{sep}{j}" + (f" {rng.random():.3f}" if values else ""))
    lines.append("% trailing comment")
    nl = "\r\n" if crlf else "\n"
    return (nl.join(lines) + (nl if rng.random() < 0.5 else "")).encode()


def test_matrix_market_device_tokenizer(tc, oracle, cuda_ok):
    """tc_graph_load_matrix_market (entries tokenized on the GPU) == host
    parse_matrix_market + build_graph, on well-formed texts with comments,
    blank lines, tabs, CRLF and value columns."""
    rng = np.random.default_rng(3)
    for k in range(12):
        n, m = int(rng.integers(5, 3000)), int(rng.integers(0, 20000))
        text = _mm_text(rng, n, m, crlf=k % 2 == 1, values=k % 3 == 0, comments=k % 4 != 0)
        el = tc.parse_matrix_market(text)
        rep_h, rep_d = tc.BuildReport(), tc.BuildReport()
        gh = tc.build_graph(el, rep_h)
        gd = tc.load_matrix_market(text, rep_d)
        assert gd.num_vertices() == gh.num_vertices() and gd.num_edges() == gh.num_edges()
        assert (rep_d.self_loops_removed, rep_d.duplicate_entries_removed) == \
               (rep_h.self_loops_removed, rep_h.duplicate_entries_removed)
        ro_h, nb_h = gh.export_csr()
        ro_d, nb_d = gd.export_csr()
        assert np.array_equal(ro_h, ro_d) and np.array_equal(nb_h, nb_d)


MM_BAD = [
    b"%%MatrixMarket matrix coordinate\n3 3 2\n1 2\n",                        # too few entries
    b"%%MatrixMarket matrix coordinate\n3 3 1\n1 x\n",                        # non-integer
    b"%%MatrixMarket matrix coordinate\n3 3 1\n1\n",                          # one token
    b"%%MatrixMarket matrix coordinate\n3 3 1\n0 1\n",                        # 1-based range
    b"%%MatrixMarket matrix coordinate\n3 3 1\n1 4\n",                        # column range
    b"%%MatrixMarket matrix coordinate\n3 3 1\n-1 2\n",                       # sign
    b"%%MatrixMarket matrix coordinate\n3 3 1\n1 2\n2 3\n",                   # content after nnz
    b"%%MatrixMarket matrix coordinate\n3 3 1\n1 2\n\n% ok\nfoo\n",           # content after nnz
    b"%%MatrixMarket matrix coordinate\n3 3 2\n1 2\n99999999999999999999 1\n",  # u64 overflow
    b"%%MatrixMarket matrix coordinate\n3 3 0\n1 2\n",                        # nnz = 0 then content
    b"%%MatrixMarket matrix coordinate\n3 3 2\n% c\n1 2\n  \n2 3x\n",         # trailing garbage
]


def test_matrix_market_device_errors(tc, cuda_ok):
    """Malformed texts raise the host parser's ParseError (same message and
    line) through the device loader."""
    for text in MM_BAD:
        with pytest.raises(tc.ParseError) as eh:
            tc.parse_matrix_market(text)
        with pytest.raises(tc.ParseError) as ed:
            tc.load_matrix_market(text)
        assert str(ed.value) == str(eh.value) and ed.value.line == eh.value.line, text
    g = tc.load_matrix_market(b"%%MatrixMarket matrix coordinate\n3 3 3\n1 2\n2 3\n3 1\n% end\n")
    assert tc.count_triangles(g).count == 1
    g0 = tc.load_matrix_market(b"%%MatrixMarket matrix coordinate\n4 4 0\n% nothing\n")
    assert g0.num_vertices() == 4 and g0.num_edges() == 0 and tc.count_triangles(g0).count == 0


def _check_listings(rows, off, nb, T):
    """rows = all T triangles exactly once: ascending, distinct, all closed."""
    assert rows.shape == (T, 3)
    if T == 0:
        return
    assert np.all(rows[:, 0] < rows[:, 1]) and np.all(rows[:, 1] < rows[:, 2])
    key = (rows[:, 0].astype(np.uint64) << np.uint64(42)) | (rows[:, 1].astype(np.uint64) << np.uint64(21)) | \
        rows[:, 2].astype(np.uint64)
    assert np.unique(key).size == T

    def has(a, b):
        seg = nb[off[a]:off[a + 1]]
        i = np.searchsorted(seg, b)
        return i < seg.size and seg[i] == b
    for a, b, c in rows[:: max(1, T // 2000)]:
        assert has(a, b) and has(a, c) and has(b, c)


def test_listings(tc, oracle, cuda_ok):
    """keep_listings (matcher.hpp:92): every triangle once, ids ascending --
    on random G(n,p), an RMAT graph and a clique (all rows checked closed on
    the small graphs)."""
    rng = np.random.default_rng(17)
    for i in range(40):
        n = int(rng.integers(20, 201))
        p = (0.02, 0.1, 0.3)[i % 3]
        iu, ju = np.triu_indices(n, 1)
        keep = rng.random(iu.size) < p
        pairs = np.stack([iu[keep], ju[keep]], 1).astype(np.uint32).reshape(-1)
        off, nb, E, _, _ = oracle.build_graph(pairs, n)
        T, pv = oracle.count(off, nb, per_vertex=True)
        r = tc.count_triangles(tc.build_graph_from_pairs(pairs, n), tc.MatchOptions(keep_listings=True))
        assert r.count == T
        _check_listings(r.listings, off, nb, T)
        hist = np.bincount(r.listings.reshape(-1), minlength=n).astype(np.uint64)
        assert np.array_equal(hist, pv)
    pairs = tc.generate(tc.GEN_RMAT, 13, 16)
    off, nb, E, _, _ = oracle.build_graph(pairs, 1 << 13)
    T, pv = oracle.count(off, nb, per_vertex=True)
    rows = tc.list_triangles(tc.build_graph_from_pairs(pairs, 1 << 13))
    _check_listings(rows, off, nb, T)
    assert np.array_equal(np.bincount(rows.reshape(-1), minlength=1 << 13).astype(np.uint64), pv)


def test_listings_streamed(tc, oracle, cuda_ok):
    """Streamed listings (tc_list_triangles_range / iter_listings): edge ranges
    partition the listing, and a bounded buffer (host or device) walks the
    whole RMAT s13 graph; the concatenated chunks equal the full listing."""
    import torch
    pairs = tc.generate(tc.GEN_RMAT, 13, 16)
    off, nb, E, _, _ = oracle.build_graph(pairs, 1 << 13)
    T, pv = oracle.count(off, nb, per_vertex=True)
    g = tc.build_graph_from_pairs(pairs, 1 << 13)
    Eo = g.num_edges()
    cuts = [0, 1, 17, Eo // 3, Eo // 3, Eo - 5, Eo]
    parts = [tc.list_triangles(g, a, b) for a, b in zip(cuts, cuts[1:])]
    assert sum(p.shape[0] for p in parts) == T
    _check_listings(np.concatenate(parts), off, nb, T)
    for cap in (1000, 50000):
        chunks = [c.copy() for c in tc.iter_listings(g, max_rows=cap)]
        assert all(0 < c.shape[0] <= cap for c in chunks)
        rows = np.concatenate(chunks)
        _check_listings(rows, off, nb, T)
        assert np.array_equal(np.bincount(rows.reshape(-1), minlength=1 << 13).astype(np.uint64), pv)
    dev = torch.empty((4096, 3), dtype=torch.int32, device="cuda")
    rows = np.concatenate([c.cpu().numpy().view(np.uint32) for c in tc.iter_listings(g, max_rows=4096, out=dev)])
    _check_listings(rows, off, nb, T)
    with pytest.raises(tc.InvalidArgument):
        tc.list_triangles(g, 5, 3)
    with pytest.raises(tc.InvalidArgument):
        tc.list_triangles(g, 0, Eo + 1)


def test_csr_route_input_residency(tc, oracle, cuda_ok):
    """tc_graph_from_csr with the CSR on the device, on the host (pageable and
    pinned, streamed in pieces) and mixed: identical graphs and counts."""
    import torch
    pairs = tc.generate(tc.GEN_RMAT, 14, 16)
    off, nb, E, _, _ = oracle.build_graph(pairs, 1 << 14)
    T, pv = oracle.count(off, nb, per_vertex=True)
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    d_nb = torch.from_numpy(nb.view(np.int32)).cuda()
    p_off = torch.from_numpy(off.view(np.int64)).pin_memory()
    p_nb = torch.from_numpy(nb.view(np.int32)).pin_memory()
    os.environ["TCB_FEED_CHUNK"] = "100000"
    try:
        for o, b in ((d_off, d_nb), (off, nb), (p_off, p_nb), (off, d_nb), (d_off, nb)):
            g = tc.graph_from_csr(o, b, 1 << 14, E)
            r = _count(tc, g)
            assert r.count == T and np.array_equal(r.per_vertex, pv)
            ro, nbr = g.export_csr()
            assert np.array_equal(ro, off) and np.array_equal(nbr, nb)
    finally:
        os.environ.pop("TCB_FEED_CHUNK", None)


def test_csr_route_errors_streamed(tc, oracle, cuda_ok):
    """Validation failures while the neighbour array is still streaming in
    (bad offsets fail before any row is oriented, bad ids after): the call
    raises, no copy outlives it, and the next build is clean."""
    pairs = tc.generate(tc.GEN_RMAT, 12, 16)
    off, nb, E, _, _ = oracle.build_graph(pairs, 1 << 12)
    T = oracle.count(off, nb)
    os.environ["TCB_FEED_CHUNK"] = "5000"
    try:
        bad_off = off.copy()
        bad_off[7] = bad_off[8] + 1  # non-monotone
        with pytest.raises(tc.InvalidArgument):
            tc.graph_from_csr(bad_off, nb, 1 << 12, E)
        bad_nb = nb.copy()
        bad_nb[len(nb) - 3] = 1 << 20  # out of range, in the last piece
        with pytest.raises(tc.InvalidArgument):
            tc.graph_from_csr(off, bad_nb, 1 << 12, E)
        assert tc.count_triangles(tc.graph_from_csr(off, nb, 1 << 12, E)).count == T
    finally:
        os.environ.pop("TCB_FEED_CHUNK", None)


def test_csr_route_empty_and_isolated(tc, cuda_ok):
    """Graph(n, 0, offsets, {}) and graphs with isolated vertices through the
    CSR route (host and streamed)."""
    for n in (0, 1, 5):
        g = tc.graph_from_csr(np.zeros(n + 1, np.uint64), np.zeros(0, np.uint32), n, 0)
        assert g.num_edges() == 0 and tc.count_triangles(g).count == 0
        r = tc.count_triangles(g, tc.MatchOptions(per_vertex=True))
        assert r.count == 0 and (r.per_vertex is None or not r.per_vertex.any())
    # K3 on vertices {2, 5, 7} of 10, the rest isolated
    off = np.array([0, 0, 0, 2, 2, 2, 4, 4, 6, 6, 6], np.uint64)
    nb = np.array([5, 7, 2, 7, 2, 5], np.uint32)
    os.environ["TCB_FEED_CHUNK"] = "2"
    try:
        r = tc.count_triangles(tc.graph_from_csr(off, nb), tc.MatchOptions(per_vertex=True))
    finally:
        os.environ.pop("TCB_FEED_CHUNK", None)
    assert r.count == 1 and r.per_vertex.tolist() == [0, 0, 1, 0, 0, 1, 0, 1, 0, 0]


@pytest.mark.slow
def test_c5_rmat_s26(tc, oracle, cuda_ok):
    """BASELINE configs[4] (RMAT s26 ef32, 2.08e9 edges) on one GPU: build
    report against SURVEY 8 / the big golden, the count against the
    independent listing kernel (listing.cu: per-edge binary searches, no
    in-edge index, no bitmap join) and, once generated, against the
    tests/golden big-config checker (oracle/big_golden, T and per-vertex)."""
    import torch
    syn = load_golden("synthetic.json")
    c = syn.get("C5_rmat_s26_ef32")
    m = tc.gen_num_edges(tc.GEN_RMAT, 26, 32)
    d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
    tc.generate(tc.GEN_RMAT, 26, 32, out=d)
    rep = tc.BuildReport()
    g = tc.build_graph_from_pairs(d, 1 << 26, rep, m=m)
    del d
    torch.cuda.empty_cache()
    # SURVEY.md section 8 config table
    assert (g.num_edges(), rep.self_loops_removed, rep.duplicate_entries_removed) == (2078632673, 8492, 68842483)
    T = tc.count_triangles(g).count
    assert tc.list_triangles_count(g) == T
    if c is not None:
        assert T == c["T"]
        try:
            r = tc.count_triangles(g, tc.MatchOptions(per_vertex=True))
        except MemoryError:
            pytest.skip("per-vertex masks of C5 do not fit next to the graph on this device")
        assert r.count == T
        assert oracle.fnv(r.per_vertex) == c["pv_fnv"]
        assert int(r.per_vertex.sum()) == 3 * T


@pytest.mark.slow
def test_rmat_s26_ef34_beyond_2p32_entries(tc, cuda_ok):
    """RMAT s26 ef34: 2.28e9 raw pairs, a symmetric CSR of more than 2^32
    directed entries (graph.hpp:64's u64 row offsets; ef32 = C5 stays just
    below).  Build report consistent, the count equal to the independent
    listing kernel, per-vertex summing to 3T; the u64-offset CSR exported on
    the device and re-ingested through the tc_graph_from_csr route gives the
    same graph and count."""
    import torch
    m = tc.gen_num_edges(tc.GEN_RMAT, 26, 34)
    n = 1 << 26
    d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
    tc.generate(tc.GEN_RMAT, 26, 34, out=d)
    rep = tc.BuildReport()
    g = tc.build_graph_from_pairs(d, n, rep, m=m)
    del d
    torch.cuda.empty_cache()
    E = g.num_edges()
    assert 2 * E >= 1 << 32
    assert rep.self_loops_removed + rep.duplicate_entries_removed + E == m
    T = tc.count_triangles(g).count
    assert tc.list_triangles_count(g) == T
    deg = torch.from_numpy(tc.degrees(g).astype(np.int64)).cuda()
    ro = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    nb = torch.empty(2 * E, dtype=torch.int32, device="cuda")
    g.export_csr(ro, nb)
    assert int(ro[-1]) == 2 * E and int(ro[0]) == 0
    assert torch.equal(ro[1:] - ro[:-1], deg)
    del g, deg
    tc.release_cached_memory()
    torch.cuda.empty_cache()
    g2 = tc.graph_from_csr(ro, nb, n, E)
    del ro, nb
    torch.cuda.empty_cache()
    assert g2.num_edges() == E
    assert tc.count_triangles(g2).count == T
    tc.release_cached_memory()
    try:
        r = tc.count_triangles(g2, tc.MatchOptions(per_vertex=True))
    except MemoryError:
        pytest.skip("per-vertex masks of this graph do not fit next to it on this device")
    assert r.count == T and int(r.per_vertex.sum()) == 3 * T
    del g2
    tc.release_cached_memory()
    torch.cuda.empty_cache()


def test_count_cuda_graph_replay(tc, oracle, cuda_ok):
    """A whole count (plan + joins + row pass + outputs) captured once into a
    CUDA graph and replayed (bench.py's timed steps): no host sync, no
    allocation inside the capture, results identical to direct launches."""
    import torch
    c = load_golden("synthetic.json")["C1_rmat_s16_ef16"]
    pairs = tc.generate(tc.GEN_RMAT, 16, 16)
    g = tc.build_graph_from_pairs(pairs, c["n"])
    st = torch.cuda.Stream()
    g.set_stream(st.cuda_stream)
    with torch.cuda.stream(st):
        tot = torch.zeros(1, dtype=torch.int64, device="cuda")
        pv = torch.zeros(c["n"], dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    opts = tc.MatchOptions(per_vertex=True)
    tc.count_triangles_into(g, tot, pv, opts)  # warm-up: scratch sized outside the capture
    torch.cuda.synchronize()
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg, stream=st, capture_error_mode="relaxed"):
        tc.count_triangles_into(g, tot, pv, opts)
    for _ in range(3):
        with torch.cuda.stream(st):
            tot.zero_()
            pv.zero_()
            cg.replay()
        torch.cuda.synchronize()
        assert int(tot.item()) == c["T"]
        assert oracle.fnv(pv.cpu().numpy().view(np.uint64)) == c["pv_fnv"]


def test_pageable_bounce_copies(tc, oracle, cuda_ok):
    """Large pageable host buffers go through the pinned bounce slots (feed.cu
    copy_h2d / copy_d2h, >= 16 MB): exported CSR arrays, re-ingested offsets and
    per-vertex counts equal the pinned-memory path byte for byte."""
    import torch
    c = load_golden("synthetic.json")["C2_er_s20_d32"]
    g = tc.build_graph_from_pairs(tc.generate(tc.GEN_ER, 20, 32), c["n"])
    n, E = c["n"], g.num_edges()
    ro_p = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    nb_p = torch.empty(2 * E, dtype=torch.int32, pin_memory=True)
    g.export_csr(ro_p, nb_p)
    ro, nb = g.export_csr()  # numpy (pageable): the 134 MB neighbour array takes the bounce path
    assert nb.nbytes >= 16 << 20
    assert np.array_equal(ro, ro_p.numpy().view(ro.dtype)) and np.array_equal(nb, nb_p.numpy().view(nb.dtype))
    assert oracle.fnv(ro) == c["offsets_fnv"] and oracle.fnv(nb) == c["nbrs_fnv"]
    # re-ingested from the pageable arrays; the large-offsets (H2D) and
    # per-vertex (D2H) bounce legs are pinned by the C3 golden (n = 2^22: 33.5 MB each)
    g2 = tc.graph_from_csr(ro, nb)
    r = tc.count_triangles(g2, tc.MatchOptions(per_vertex=True))
    assert r.count == c["T"] and int(r.per_vertex.sum()) == 3 * c["T"]


def test_pageable_bounce_large_n(tc, oracle, cuda_ok):
    """C1's edges in a graph declared with n = 2^22 ids: the offsets (33.5 MB)
    exported to and re-ingested from pageable numpy arrays, and the per-vertex
    counts (33.5 MB) read back into one, all through the bounce slots; the
    counts equal the C1 golden and the extra ids count zero."""
    c = load_golden("synthetic.json")["C1_rmat_s16_ef16"]
    n = 1 << 22
    g = tc.build_graph_from_pairs(tc.generate(tc.GEN_RMAT, 16, 16), n)
    ro, nb = g.export_csr()
    assert ro.nbytes >= 16 << 20 and ro.shape[0] == n + 1 and int(ro[-1]) == 2 * c["E"]
    g2 = tc.graph_from_csr(ro, nb)
    r = tc.count_triangles(g2, tc.MatchOptions(per_vertex=True))
    assert r.per_vertex.nbytes >= 16 << 20
    assert r.count == c["T"]
    assert oracle.fnv(np.ascontiguousarray(r.per_vertex[:c["n"]])) == c["pv_fnv"]
    assert not r.per_vertex[c["n"]:].any()
