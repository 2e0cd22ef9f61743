"""Summarise an ncu report: key SOL/memory/warp metrics + top SASS lines by stall samples."""
import re
import csv, subprocess, sys, io
rep = sys.argv[1]; kern = sys.argv[2] if len(sys.argv) > 2 else ""
nlines = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]; ki, si, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Value", "Metric Unit"))
want = {"Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput",
        "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Issue Slots Busy", "Executed Ipc Active",
        "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp", "Achieved Occupancy",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Grid Size", "Mem Pipes Busy"}
for x in r[1:]:
    if re.search(kern, x[ki]) and x[mi] in want:
        print(f"  {x[mi]:45s} {x[vi]:>14s} {x[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
             "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_sector_hit_rate.pct", "sm__inst_executed.sum"):
    if name in hh:
        j = hh.index(name)
        for row in rr[2:]:
            if re.search(kern, row[hh.index("Kernel Name")]):
                print(f"  {name:45s} {row[j]:>14s} {rr[1][j]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern or '.'}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = [i for i, x in enumerate(rows) if "Address" in x and "Source" in x][0]
h = rows[hi]
I = h.index
data = []
for x in rows[hi + 1:]:
    try:
        data.append((int(x[I("Warp Stall Sampling (All Samples)")]), int(x[I("Instructions Executed")]),
                     float(x[I("Avg. Threads Executed")]), x[I("Address")][-5:], x[I("Source")].strip()))
    except Exception:
        pass
tot = sum(d[0] for d in data) or 1; toti = sum(d[1] for d in data) or 1
print(f"  samples={tot} warp-inst={toti}")
for d in sorted(data, key=lambda d: -d[0])[:nlines]:
    print(f"  {100*d[0]/tot:5.1f}% {100*d[1]/toti:5.1f}%i thr={d[2]:5.1f} {d[3]} {d[4][:80]}")

# aggregated stall reasons
idx = [(j, nm) for j, nm in enumerate(h) if nm.startswith("stall_") and "(Not Issued)" not in nm]
agg = {}
for x in rows[hi + 1:]:
    for j, nm in idx:
        try:
            agg[nm] = agg.get(nm, 0) + float(x[j])
        except Exception:
            pass
T = sum(agg.values()) or 1
print("  stall reasons: " + ", ".join(f"{k[6:]}={100*v/T:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
