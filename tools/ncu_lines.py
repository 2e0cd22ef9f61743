"""Per-CUDA-source-line stall samples and executed instructions of one kernel
from an ncu report (--print-source cuda,sass): python tools/ncu_lines.py rep kernel_regex [n]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
fname = ""
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0]:
        continue
    try:
        smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        ins = int(r[hdr.index("Instructions Executed")])
    except ValueError:
        continue
    key = (fname, int(r[0]))
    a = agg.setdefault(key, [0, 0, r[1].strip()[:90]])
    a[0] += smp
    a[1] += ins
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
print(f"samples={ts} warp-inst={ti}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100*a[0]/ts:5.1f}%s {100*a[1]/ti:5.1f}%i {k[0]}:{k[1]:<5d} {a[2]}")
