"""CPU: pin the oracle (oracle/oracle.c) against the reference's own golden
vectors (tests/golden/, generated from oracle/_ref by make_golden.py) and, when
oracle/_ref is built, against the reference library directly."""
import numpy as np
import pytest

from conftest import load_golden


def _pairs(case):
    return np.array(case.get("pairs", case.get("edges", [])), dtype=np.uint32).reshape(-1)


def test_known_answers(oracle):
    known = load_golden("known.json")
    for name, c in known.items():
        if name.startswith("_") or c.get("skip_ref_csr"):
            continue
        off, nb, E, lo, du = oracle.build_graph(_pairs(c), c["n"])
        assert (E, lo, du) == (c["E"], c["loops"], c["dups"]), name
        assert off.tolist() == c["offsets"], name
        assert nb.tolist() == c["nbrs"], name
        T, pv = oracle.count(off, nb, per_vertex=True)
        assert T == c["T"], name
        assert pv.tolist() == c["per_vertex"], name
        if c["n"] <= 5000:
            assert oracle.brute_force(off, nb) == T, name


def test_spec_examples(oracle):
    # SPEC.md:63-65 / :292-294 / :308 / :317-318 / :363-364
    expect = {"K3": 1, "K4": 4, "K5": 10, "star_S4": 0, "path_P3": 0, "empty": 0}
    known = load_golden("known.json")
    for k, t in expect.items():
        assert known[k]["T"] == t
    assert known["K3"]["offsets"] == [0, 2, 4, 6] and known["K3"]["nbrs"] == [1, 2, 0, 2, 0, 1]
    assert known["loop_mirror_2"]["E"] == 1 and known["loop_mirror_2"]["nbrs"] == [1, 0]


def test_out_of_range(oracle):
    with pytest.raises(ValueError):
        oracle.build_graph(np.array([0, 5], np.uint32), 3)
    assert load_golden("known.json")["_out_of_range"]["error_code"] == 1


def test_gnp_golden(oracle):
    for i, c in enumerate(load_golden("gnp.json")):
        off, nb, E, lo, du = oracle.build_graph(_pairs(c), c["n"])
        assert (E, lo, du) == (c["E"], c["loops"], c["dups"]), i
        T, pv = oracle.count(off, nb, per_vertex=True)
        assert T == c["T"], i
        assert pv.tolist() == c["per_vertex"], i


def test_gnp_500_brute_force(oracle):
    # SPEC.md:438-446 acceptance: >=500 random G(n<=200, p in {.02,.1,.3})
    rng = np.random.default_rng(7)
    for i in range(510):
        n = int(rng.integers(20, 201))
        p = (0.02, 0.1, 0.3)[i % 3]
        iu, ju = np.triu_indices(n, 1)
        keep = rng.random(iu.size) < p
        pairs = np.stack([iu[keep], ju[keep]], 1).astype(np.uint32).reshape(-1)
        off, nb, E, _, _ = oracle.build_graph(pairs, n)
        assert oracle.count(off, nb) == oracle.brute_force(off, nb)


def test_generator_fingerprints(oracle):
    syn = load_golden("synthetic.json")
    for name, c in syn.items():
        if c["m"] > (1 << 22):
            continue
        if c["kind"] == "er":
            pairs = oracle.gen_er(c["scale"], c["edgefactor"])
        else:
            pairs = oracle.gen_rmat(c["scale"], c["edgefactor"], c["permute"])
        assert oracle.fnv(pairs) == c["pairs_fnv"], name


@pytest.mark.parametrize("name", ["C1_rmat_s16_ef16", "kron_s18_ef16"])
def test_synthetic_golden(oracle, name):
    c = load_golden("synthetic.json")[name]
    pairs = oracle.gen_rmat(c["scale"], c["edgefactor"], c["permute"])
    off, nb, E, lo, du = oracle.build_graph(pairs, c["n"])
    assert (E, lo, du) == (c["E"], c["loops"], c["dups"])
    assert oracle.fnv(off) == c["offsets_fnv"] and oracle.fnv(nb) == c["nbrs_fnv"]
    T, pv = oracle.count(off, nb, per_vertex=True)
    assert T == c["T"]
    assert oracle.fnv(pv) == c["pv_fnv"]


def test_survey_numbers(oracle):
    # SURVEY.md section 8 config table (splitmix generator)
    syn = load_golden("synthetic.json")
    assert syn["C1_rmat_s16_ef16"]["E"] == 909250 and syn["C1_rmat_s16_ef16"]["T"] == 15608808
    assert syn["C1_rmat_s16_ef16"]["loops"] == 497 and syn["C1_rmat_s16_ef16"]["dups"] == 138829
    assert syn["C2_er_s20_d32"]["E"] == 16776954 and syn["C2_er_s20_d32"]["T"] == 5477
    assert syn["rmat_s20_ef16"]["T"] == 424205046


def test_oracle_vs_reference_random(oracle, ref):
    rng = np.random.default_rng(11)
    for i in range(40):
        n = int(rng.integers(1, 300))
        m = int(rng.integers(0, 4 * n))
        pairs = rng.integers(0, n, 2 * m).astype(np.uint32)
        a = oracle.build_graph(pairs, n)
        b = ref.build_graph(pairs, n)
        assert a[2:] == b[2:]
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        g = ref.graph(b[0], b[1])
        T, pv = g.count_triangles(per_vertex=True)
        oT, opv = oracle.count(a[0], a[1], per_vertex=True)
        assert T == oT and np.array_equal(pv, opv)


# ---- the degree-ordered DAG checker (oracle_count_dag): pinned before it is
# trusted for the configs the id-order restatement cannot finish (C5) ----

def test_dag_checker_known_and_gnp(oracle):
    for name, c in load_golden("known.json").items():
        if name.startswith("_") or c.get("skip_ref_csr"):
            continue
        off, nb, E, lo, du = oracle.build_graph(_pairs(c), c["n"])
        T, pv = oracle.count_dag(off, nb, per_vertex=True)
        assert T == c["T"] and pv.tolist() == c["per_vertex"], name
    for i, c in enumerate(load_golden("gnp.json")):
        off, nb, E, lo, du = oracle.build_graph(_pairs(c), c["n"])
        T, pv = oracle.count_dag(off, nb, per_vertex=True)
        assert T == c["T"] and pv.tolist() == c["per_vertex"], i


@pytest.mark.parametrize("name", ["C1_rmat_s16_ef16", "kron_s18_ef16", "rmat_s18_ef16", "C2_er_s20_d32"])
def test_dag_checker_synthetic_goldens(oracle, name):
    """Against the reference's segmented_intersect goldens (T and per-vertex)."""
    c = load_golden("synthetic.json")[name]
    pairs = oracle.gen_er(c["scale"], c["edgefactor"]) if c["kind"] == "er" else \
        oracle.gen_rmat(c["scale"], c["edgefactor"], c["permute"])
    off, nb, E, lo, du = oracle.build_graph(pairs, c["n"])
    T, pv = oracle.count_dag(off, nb, per_vertex=True)
    assert T == c["T"]
    assert oracle.fnv(pv) == c["pv_fnv"]


def test_dag_checker_vs_reference_random(oracle, ref):
    rng = np.random.default_rng(5)
    for i in range(40):
        n = int(rng.integers(1, 400))
        m = int(rng.integers(0, 6 * n))
        pairs = rng.integers(0, n, 2 * m).astype(np.uint32)
        off, nb, E, _, _ = ref.build_graph(pairs, n)
        T, pv = ref.graph(off, nb).count_triangles(per_vertex=True)
        dT, dpv = oracle.count_dag(off, nb, per_vertex=True)
        assert T == dT and np.array_equal(pv, dpv)


def test_big_golden_driver_matches_c1(oracle):
    """oracle/big_golden (the streamed build + checker used for C4 per-vertex
    and C5) reproduces the C1 golden end to end."""
    import json
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "oracle", "_ref", "big_golden")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/big_golden not built")
    c = load_golden("synthetic.json")["C1_rmat_s16_ef16"]
    for mode in ("dag", "oracle"):
        out = json.loads(subprocess.run([exe, "rmat", "16", "16", mode], capture_output=True, text=True,
                                        check=True).stdout)
        for k in ("pairs_fnv", "E", "loops", "dups", "offsets_fnv", "nbrs_fnv", "T", "pv_fnv"):
            assert out[k] == c[k], (mode, k)
