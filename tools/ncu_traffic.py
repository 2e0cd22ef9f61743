"""Per-kernel DRAM traffic of one count, stamped with the library build.

  ncu --set full ... -o gpurun_out/prof_C4 python tools/prof_count.py ...
  python tools/ncu_traffic.py gpurun_out/prof_C4.ncu-rep C4

Reads dram__bytes_read.sum + dram__bytes_write.sum and gpu__time_duration.sum
of every kernel in the report (per launch; the last launch of each kernel
name wins) and writes ncu_traffic_<config>.json next to the report (copy it to profiles/) with the sha256 of
paper_1909_02127_b200/libtcb200.so.  bench.py reports `roofline.traffic` only
when that hash matches the library it runs (otherwise traffic = null).
"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_inputs_sha256(root):
    """sha256 over the library's build inputs (csrc sources, headers,
    Makefile, include/): the same sources build the same kernels, while the
    .so itself is not byte-reproducible across clean builds."""
    import hashlib
    h = hashlib.sha256()
    for d in (os.path.join(root, "paper_1909_02127_b200", "csrc"), os.path.join(root, "include")):
        for name in sorted(os.listdir(d)):
            if name.endswith((".cu", ".cuh", ".h", ".hpp", ".cpp")) or name == "Makefile":
                h.update(name.encode())
                with open(os.path.join(d, name), "rb") as f:
                    h.update(f.read())
    return h.hexdigest()


def main():
    rep, config = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
             "msecond": 1.0, "second": 1e3}
    out = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        short = name.split("(")[0].split("::")[-1].split("<")[0].strip()
        if name.startswith("void "):
            short = name[5:].split("(")[0].split("::")[-1].split("<")[0].strip()

        def val(m):
            j = h.index(m)
            return float(r[j].replace(",", "")) * scale.get(units[j], 1)
        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        out[short] = {"dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
                      "ms": val("gpu__time_duration.sum"),
                      "l2_hit_pct": val("lts__t_sector_hit_rate.pct") if "lts__t_sector_hit_rate.pct" in h else None,
                      "kernel": name[:120]}
    with open(os.path.join(ROOT, "paper_1909_02127_b200", "libtcb200.so"), "rb") as f:
        sha = hashlib.sha256(f.read()).hexdigest()
    git = os.environ.get("GIT_HEAD") or subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"],
                                                       capture_output=True, text=True).stdout.strip()
    doc = {"config": config, "lib_sha256": sha, "src_sha256": build_inputs_sha256(ROOT), "git_head": git or None,
           "report": os.path.basename(rep),
           "kernels": out}
    # written next to the report (gpurun_out/ travels back); copy it into
    # profiles/ to make bench.py use it
    path = os.path.join(os.path.dirname(os.path.abspath(rep)), f"ncu_traffic_{config}.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
