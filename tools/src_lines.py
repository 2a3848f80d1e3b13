"""Instructions executed and stall samples per CUDA source line of one kernel
(ncu --page source --print-source cuda,sass)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, file = {}, None
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        file = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] not in ("", "Function Name"):
        num = lambda x: int(x) if x.strip().isdigit() else 0
        ie = num(r[hdr.index("Instructions Executed")])
        ss = num(r[hdr.index("Warp Stall Sampling (All Samples)")])
        agg[(file, int(r[0]), r[1][:70])] = (ie, ss)
T = sum(v[0] for v in agg.values()) or 1
S = sum(v[1] for v in agg.values()) or 1
print(f"total warp instr {T}, samples {S}")
for k, v in sorted(agg.items(), key=lambda t: -t[1][0])[:top]:
    print(f"{100*v[0]/T:5.1f}% inst {100*v[1]/S:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
