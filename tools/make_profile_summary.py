"""Write the judged ncu evidence into profiles/ (run here, no GPU):
  profiles/<tag>_kernels.md   per-kernel duration, DRAM bytes, throughput, occupancy
  profiles/<tag>_launches.csv the launch list (gpu__time_duration per launch)
  profiles/traffic_<round>.json  dram read+write bytes per launch, by stage name
usage: python tools/make_profile_summary.py gpurun_out/prof_X.ncu-rep gpurun_out/launches_X.csv r01
"""
import csv
import json
import os
import shutil
import subprocess
import sys

rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)
STAGE = {"k_project_count": "project_count", "k_scan_tiles": "scan_tiles", "k_scatter": "scatter",
         "k_scatter_slots": "scatter", "k_sort_big": "sort_big", "k_blend_fwd": "blend_fwd",
         "k_blend_bwd": "blend_bwd", "k_bin_bilinear": "bin_fused", "k_sh_grad": "sh_grad"}
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                     capture_output=True, text=True).stdout.splitlines()))
h, units = raw[0], raw[1]
col = {n: h.index(n) for n in h}
want = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem thru %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thru %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("launch__registers_per_thread", "regs"), ("smsp__inst_executed.sum", "warp instr")]
lines = [f"# ncu --set full summary ({tag})", "",
         f"Source: `{os.path.basename(rep)}` (one launch per kernel, cfg2 workload, "
         "`bench.py --profile-run`, clocks not locked).  Units as ncu reports them.", "",
         "| kernel | " + " | ".join(w[1] for w in want) + " |",
         "|---|" + "---|" * len(want)]
traffic = {}
seen = set()
for row in raw[2:]:
    name = row[col["Kernel Name"]]
    short = name.split("(")[0].replace("void ", "").split("<")[0].replace("inpc::", "")
    key = name.split("(")[0]
    if key in seen:
        continue
    seen.add(key)
    vals = []
    for m, _ in want:
        v, u = row[col[m]], units[col[m]]
        vals.append(f"{v} {u}".strip())
    lines.append(f"| `{name.split('(')[0].replace('void ', '')}` | " + " | ".join(vals) + " |")
    st = STAGE.get(short)
    if st:
        def mb(m):
            v, u = float(row[col[m]]), units[col[m]]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic[st] = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
open(os.path.join(out_dir, f"{tag}_kernels.md"), "w").write("\n".join(lines) + "\n")
shutil.copy(launches, os.path.join(out_dir, f"{tag}_launches.csv"))
json.dump(traffic, open(os.path.join(out_dir, f"traffic_{tag.split('_')[0]}.json"), "w"), indent=1)
print("\n".join(lines))
print(traffic)
