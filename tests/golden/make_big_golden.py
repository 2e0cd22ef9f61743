"""Big-config goldens (C4 per-vertex from the reference, C5) via oracle/big_golden.

Run in the build container (needs oracle/_ref, built from /root/reference):
    python tests/golden/make_big_golden.py c4_ref   # reference segmented_intersect + listings, ~25 min / 8 cores
    python tests/golden/make_big_golden.py c5_dag   # degree-ordered checker (pinned by tests/test_oracle.py), ~1 h
    python tests/golden/make_big_golden.py merge <json>...  # fold driver outputs into synthetic.json

big_golden streams the SURVEY 8d generator twice (degree count, scatter),
builds the symmetric CSR exactly as build_graph does (graph.cpp:33-85) and
counts with the selected checker; its output JSON carries the same keys as
synthetic.json.  The raw driver outputs used for the committed goldens are
kept next to this file (big_golden_*.json).
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
EXE = os.path.join(ROOT, "oracle", "_ref", "big_golden")
RUNS = {
    "c4_ref": ("C4_rmat_s24_ef16", ["rmat", "24", "16", "ref", "8"]),
    "c5_dag": ("C5_rmat_s26_ef32", ["rmat", "26", "32", "dag", "8"]),
}


def merge(paths):
    syn_path = os.path.join(HERE, "synthetic.json")
    syn = json.load(open(syn_path))
    for p in paths:
        d = json.load(open(p))
        name = {("rmat", 24, 16): "C4_rmat_s24_ef16", ("rmat", 26, 32): "C5_rmat_s26_ef32"}[
            (d["kind"], d["scale"], d["edgefactor"])]
        cur = syn.get(name, {})
        for k in ("kind", "scale", "edgefactor", "permute", "n", "m", "pairs_fnv", "E", "loops", "dups", "offsets_fnv",
                  "nbrs_fnv", "T", "pv_fnv", "pv_sum", "pv_max", "pv_argmax"):
            if k in cur and cur[k] != d[k]:
                raise SystemExit(f"{name}.{k}: committed {cur[k]} != {d[k]} from {p}")
            cur[k] = d[k]
        srcs = set(filter(None, [cur.get("source")]))
        srcs.add(d["source"] + f" [{os.path.basename(p)}]")
        cur["source"] = "; ".join(sorted(srcs))
        syn[name] = cur
    with open(syn_path, "w") as f:
        json.dump(syn, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    if sys.argv[1] == "merge":
        merge(sys.argv[2:])
    else:
        name, args = RUNS[sys.argv[1]]
        out = subprocess.run([EXE] + args, capture_output=True, text=True, check=True).stdout
        path = os.path.join(HERE, f"big_golden_{sys.argv[1]}.json")
        with open(path, "w") as f:
            f.write(out)
        merge([path])
