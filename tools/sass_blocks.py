"""Per-block SASS instruction / stall breakdown of one kernel in an ncu report."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
blk = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern],
                     capture_output=True, text=True).stdout
src = list(csv.reader(out.splitlines()))
hdr = src[1]
rows = [x for x in src[2:] if x and x[0].startswith("0x")]
# the page lists every profiled launch of the kernel back to back; keep the first
addr0 = rows[0][0]
for i in range(1, len(rows)):
    if rows[i][0] == addr0:
        rows = rows[:i]
        break
ie = hdr.index("Instructions Executed")
sc = hdr.index("Source")
si = hdr.index("Warp Stall Sampling (All Samples)")
totI = sum(int(x[ie] or 0) for x in rows) or 1
totS = sum(int(x[si] or 0) for x in rows) or 1
print(f"{kern}: {totI} warp-instr, {totS} stall samples, {len(rows)} SASS")
cum = 0
for b in range(0, len(rows), blk):
    bl = rows[b:b + blk]
    s = sum(int(x[ie] or 0) for x in bl)
    st = sum(int(x[si] or 0) for x in bl)
    cum += s
    ops = {}
    for x in bl:
        o = x[sc].split()
        o = o[1] if o[0].startswith("@") else o[0]
        ops[o] = ops.get(o, 0) + int(x[ie] or 0)
    top = sorted(ops.items(), key=lambda t: -t[1])[:6]
    if s or st:
        print(f"{b:5d} {100*s/totI:5.1f}% cum {100*cum/totI:5.1f}% stall {100*st/totS:5.1f}%  " +
              " ".join(f"{o}:{c//1000}k" for o, c in top))
