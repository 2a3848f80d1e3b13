"""Stall reasons per SASS region of one kernel in an ncu report."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
blk = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern],
                     capture_output=True, text=True).stdout
src = list(csv.reader(out.splitlines()))
hdr = src[1]
rows = [x for x in src[2:] if x and x[0].startswith("0x")]
a0 = rows[0][0]
for i in range(1, len(rows)):
    if rows[i][0] == a0:
        rows = rows[:i]
        break
reasons = ["stall_long_sb", "stall_short_sb", "stall_wait", "stall_math", "stall_mio", "stall_lg",
           "stall_branch_resolving", "stall_not_selected", "stall_selected", "stall_no_inst",
           "stall_dispatch", "stall_barrier", "stall_membar", "stall_drain", "stall_misc", "stall_tex"]
ci = {r: hdr.index(r) for r in reasons}
ie = hdr.index("Instructions Executed")
sc = hdr.index("Source")
tot = {r: sum(int(x[ci[r]] or 0) for x in rows) for r in reasons}
T = sum(tot.values()) or 1
print(kern, "total samples", T, {r[6:]: round(100 * v / T, 1) for r, v in sorted(tot.items(), key=lambda t: -t[1]) if v})
for b in range(0, len(rows), blk):
    bl = rows[b:b + blk]
    st = {r: sum(int(x[ci[r]] or 0) for x in bl) for r in reasons}
    s = sum(st.values())
    if s / T < 0.02:
        continue
    ins = sum(int(x[ie] or 0) for x in bl)
    ops = {}
    for x in bl:
        o = x[sc].split()
        o = o[1] if o[0].startswith("@") else o[0]
        ops[o] = ops.get(o, 0) + int(x[ie] or 0)
    top = sorted(ops.items(), key=lambda t: -t[1])[:4]
    print(f"{b:5d} {100*s/T:5.1f}% inst {ins//1000}k | " +
          " ".join(f"{r[6:]}:{100*v/T:.1f}" for r, v in sorted(st.items(), key=lambda t: -t[1])[:4] if v) +
          " | " + " ".join(f"{o}" for o, c in top))
