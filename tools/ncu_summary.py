"""Summarise an ncu report here (no GPU): per kernel duration, DRAM bytes,
throughputs, occupancy, and the top SASS stall lines."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(ncu("--page", "raw", "--csv").splitlines()))
h = raw[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
idx = [h.index(w) if w in h else None for w in want]
units = raw[1]
print(" | ".join(w.split(".")[0][-28:] for w in want))
for row in raw[2:]:
    print(" | ".join((row[i][:40] + (" " + units[i] if units[i] and j else "")) if i is not None else "-"
                     for j, i in enumerate(idx)))

names = sorted({r[h.index("Kernel Name")] for r in raw[2:]})
for n in names:
    short = n.split("(")[0].replace("void ", "")
    src = list(csv.reader(ncu("--page", "source", "--csv", "--kernel-name", "regex:" + short.split("::")[-1].split("<")[0]).splitlines()))
    if len(src) < 3:
        continue
    hdr = src[1]
    rows = [x for x in src[2:] if x and x[0].startswith("0x")]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    sc = hdr.index("Source")
    tot = sum(int(x[si] or 0) for x in rows) or 1
    totI = sum(int(x[ie] or 0) for x in rows)
    print(f"\n== {short}: {totI} warp-instr, {tot} samples")
    best = sorted(range(len(rows)), key=lambda i: -int(rows[i][si] or 0))[:top]
    for i in sorted(best):
        x = rows[i]
        print(f"  {i:5d} {100*int(x[si] or 0)/tot:5.1f}% {int(x[ie] or 0):>9} {x[sc][:80]}")
