"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference for oracle/_ref):
    python tests/golden/make_golden.py [--big]

Every expected value below comes from oracle/_ref/libtrimatch_ref.so -- the
reference's own sources (trimatch::build_graph, count_triangles,
segmented_intersect) compiled by oracle/Makefile -- never from our CUDA path.
The inputs are the deterministic generators of SURVEY.md section 8d (restated in
oracle/oracle.c); their fingerprints are stored so the device generator can be
checked bit-exactly on the GPU box without /root/reference.

Outputs:
  known.json     -- SPEC.md known answers (K3/K4/K5/star/path/empty/loops/dups)
  gnp.json       -- random G(n,p) instances (n<=200, p in {0.02,0.1,0.3}) with
                    edge lists, counts (matcher + segmented-intersect) and
                    per-vertex arrays
  synthetic.json -- C1/C2/s18/s20 (+ C3/C4 totals with --big): |E|, loops, dups,
                    T, per-vertex FNV-1a-64 / sum / max, CSR fingerprints
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle_ctypes import Oracle, Ref  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def known(ref: Ref):
    cases = {
        "K3": (3, [(0, 1), (0, 2), (1, 2)]),
        "K4": (4, [(a, b) for a in range(4) for b in range(a + 1, 4)]),
        "K5": (5, [(a, b) for a in range(5) for b in range(a + 1, 5)]),
        "star_S4": (5, [(0, i) for i in range(1, 5)]),
        "path_P3": (3, [(0, 1), (1, 2)]),
        "empty": (0, []),
        "isolated_only": (7, []),
        "K3_loop_mirror": (3, [(0, 1), (1, 0), (0, 0), (1, 2), (2, 2), (2, 0), (0, 2)]),
        "loop_mirror_2": (2, [(0, 0), (0, 1), (1, 0)]),
        "all_dups": (4, [(1, 2)] * 9),
        "all_loops": (4, [(i, i) for i in range(4)] * 3),
        "two_K4_share_edge": (6, [(a, b) for a in range(4) for b in range(a + 1, 4)]
                              + [(a, b) for a in (0, 1, 4, 5) for b in (0, 1, 4, 5) if a < b]),
        "K3_high_ids": (0xFFFFFFFF, [(0xFFFFFFFE, 0xFFFFFFFD), (0xFFFFFFFD, 7), (7, 0xFFFFFFFE)]),
    }
    out = {}
    for name, (n, edges) in cases.items():
        pairs = np.array(edges, dtype=np.uint32).reshape(-1)
        if n > 10_000_000:
            # too many declared vertices for the reference's dense arrays here;
            # only record the expected triangle structure
            out[name] = dict(n=n, edges=edges, E=3, loops=0, dups=0, T=1, skip_ref_csr=True)
            continue
        off, nb, E, lo, du = ref.build_graph(pairs, n)
        g = ref.graph(off, nb)
        T, pv = g.count_triangles(per_vertex=True)
        out[name] = dict(n=n, edges=edges, E=E, loops=lo, dups=du, T=T,
                         offsets=off.tolist(), nbrs=nb.tolist(), per_vertex=pv.tolist())
    # out-of-range ids -> std::invalid_argument (graph.cpp:40-42)
    try:
        ref.build_graph(np.array([0, 5], dtype=np.uint32), 3)
        raise SystemExit("expected invalid_argument")
    except Exception as e:  # RefError code 1
        out["_out_of_range"] = dict(n=3, edges=[(0, 5)], error_code=getattr(e, "code", None))
    return out


def gnp(ref: Ref, count: int):
    rng = np.random.default_rng(20190905)
    cases = []
    ps = [0.02, 0.1, 0.3]
    for i in range(count):
        n = int(rng.integers(20, 201))
        p = ps[i % 3]
        iu, ju = np.triu_indices(n, 1)
        keep = rng.random(iu.size) < p
        a, b = iu[keep].astype(np.uint32), ju[keep].astype(np.uint32)
        # randomise orientation, add a few loops and duplicate entries like raw input
        flip = rng.random(a.size) < 0.5
        src = np.where(flip, b, a)
        dst = np.where(flip, a, b)
        extra = int(rng.integers(0, 4))
        loops = rng.integers(0, n, extra).astype(np.uint32)
        dupi = rng.integers(0, max(a.size, 1), extra) if a.size else np.zeros(0, np.int64)
        src = np.concatenate([src, loops, dst[dupi] if a.size else []]).astype(np.uint32)
        dst = np.concatenate([dst, loops, src[dupi] if a.size else []]).astype(np.uint32)
        pairs = np.stack([src, dst], 1).reshape(-1)
        off, nb, E, lo, du = ref.build_graph(pairs, n)
        g = ref.graph(off, nb)
        T0 = g.count_triangles(lookahead=0, workers=1)
        T, pv = g.count_triangles(lookahead=2, per_vertex=True)
        Ts = g.segmented_intersect()
        assert T0 == T == Ts, (i, T0, T, Ts)
        cases.append(dict(n=n, p=p, pairs=pairs.tolist(), E=E, loops=lo, dups=du, T=T,
                          per_vertex=pv.tolist()))
    return cases


def synthetic(o: Oracle, ref: Ref, big: bool, big_only: bool = False):
    big = big or big_only
    cfgs = [] if big_only else [
        ("C1_rmat_s16_ef16", "rmat", 16, 16, False),
        ("C2_er_s20_d32", "er", 20, 32, False),
        ("rmat_s18_ef16", "rmat", 18, 16, False),
        ("kron_s18_ef16", "rmat", 18, 16, True),
        ("rmat_s20_ef16", "rmat", 20, 16, False),
    ]
    if big:
        cfgs += [("C3_kron_s22_ef16", "rmat", 22, 16, True)]
    out = {}
    for name, kind, scale, ef, perm in cfgs:
        t0 = time.time()
        pairs = o.gen_er(scale, ef) if kind == "er" else o.gen_rmat(scale, ef, perm)
        n = 1 << scale
        off, nb, E, lo, du = ref.build_graph(pairs, n)
        g = ref.graph(off, nb)
        T, pv = g.segmented_intersect(per_vertex=True)
        rec = dict(kind=kind, scale=scale, edgefactor=ef, permute=perm, n=n, m=int(pairs.size // 2),
                   pairs_fnv=o.fnv(pairs), E=E, loops=lo, dups=du, T=T,
                   offsets_fnv=o.fnv(off), nbrs_fnv=o.fnv(nb),
                   pv_fnv=o.fnv(pv), pv_sum=int(pv.sum()), pv_max=int(pv.max()),
                   pv_argmax=int(pv.argmax()), source="reference segmented_intersect (SPEC.md:376)")
        if scale <= 16:
            rec["T_count_triangles"] = g.count_triangles()
            assert rec["T_count_triangles"] == T
        out[name] = rec
        print(name, rec["E"], rec["T"], "%.1fs" % (time.time() - t0), flush=True)
    if big:
        # C4: the reference's segmented_intersect total from SURVEY.md section 8
        # (1,046.7 s at 8 workers); the per-vertex array is from oracle.c (which
        # equals the reference listing histogram on every smaller config above).
        pairs = o.gen_rmat(24, 16, False)
        off, nb, E, lo, du = o.build_graph(pairs, 1 << 24)
        T, pv = o.count(off, nb, per_vertex=True)
        assert T == 10282799137, T
        out["C4_rmat_s24_ef16"] = dict(kind="rmat", scale=24, edgefactor=16, permute=False, n=1 << 24,
                                       m=int(pairs.size // 2), pairs_fnv=o.fnv(pairs), E=E, loops=lo,
                                       dups=du, T=T, offsets_fnv=o.fnv(off), nbrs_fnv=o.fnv(nb),
                                       pv_fnv=o.fnv(pv), pv_sum=int(pv.sum()), pv_max=int(pv.max()),
                                       pv_argmax=int(pv.argmax()),
                                       source="T: reference segmented_intersect (SURVEY.md 8); "
                                              "per-vertex: oracle.c")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--gnp", type=int, default=90)
    ap.add_argument("--only", default="known,gnp,synthetic")
    ap.add_argument("--big-only", action="store_true", help="only C3/C4 (implies --big)")
    a = ap.parse_args()
    o, ref = Oracle(), Ref()
    only = a.only.split(",")
    if "known" in only:
        json.dump(known(ref), open(os.path.join(HERE, "known.json"), "w"))
    if "gnp" in only:
        json.dump(gnp(ref, a.gnp), open(os.path.join(HERE, "gnp.json"), "w"))
    if "synthetic" in only:
        path = os.path.join(HERE, "synthetic.json")
        new = synthetic(o, ref, a.big, a.big_only)
        old = json.load(open(path)) if os.path.exists(path) else {}
        old.update(new)
        json.dump(old, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
