"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel total ms."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
tot = {}
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    name = r[ki].split("(")[0][-48:]
    tot.setdefault(name, [0.0, 0]); tot[name][0] += float(r[vi].replace(",", "")) / 1e6; tot[name][1] += 1
for k, v in sorted(tot.items(), key=lambda x: -x[1][0]):
    print(f"{v[0]:10.3f} ms {v[1]:5d}  {k}")
