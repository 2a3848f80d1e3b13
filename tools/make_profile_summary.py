"""Write the judged ncu evidence into profiles/ (run here, no GPU):
  profiles/<tag>_kernels.md      per-kernel duration, DRAM bytes, throughput, occupancy, per config
  profiles/<tag>_launches.csv    the launch list (gpu__time_duration per launch, cfg 2 workload)
  profiles/traffic_<tag>.json    dram read+write bytes per launch, by config and stage name
usage: python tools/make_profile_summary.py TAG LAUNCHES.csv KEY=REPORT.ncu-rep [KEY=REPORT ...]
  KEY: cfg2, cfg3, cfg4, cfg5, cfg2-sh, cfg2-env (bench.py looks traffic up by this key)
"""
import csv
import json
import os
import shutil
import subprocess
import sys

tag, launches = sys.argv[1], sys.argv[2]
reports = [a.split("=", 1) for a in sys.argv[3:]]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_dir = os.environ.get("PROFILE_OUT", os.path.join(ROOT, "profiles"))
os.makedirs(out_dir, exist_ok=True)
STAGE = {"k_project_count": "project_count", "k_scan_tiles": "scan_tiles", "k_scatter": "scatter",
         "k_scatter_slots": "scatter", "k_sort_big": "sort_big", "k_blend_fwd": "blend_fwd",
         "k_blend_bwd": "blend_bwd", "k_bin_bilinear": "bin_fused", "k_sh_grad": "sh_grad"}
WANT = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem thru %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thru %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("launch__registers_per_thread", "regs"), ("smsp__inst_executed.sum", "warp instr")]
WORKLOAD = {"cfg2": "cfg 2 (2^20 points, 1080p, bilinear, fwd+bwd)",
            "cfg3": "cfg 3 (4x2^20 points, Gaussian, fwd)",
            "cfg4": "cfg 4 (2^25 points, bilinear, fwd, unfused binning)",
            "cfg5": "cfg 5 (64 views of 2^23 points, fwd+bwd)",
            "cfg2-sh": "cfg 2 with SH degree-2 features (f1)",
            "cfg2-env": "cfg 2 with an environment-map background (f2)"}
lines = [f"# ncu --set full summary ({tag})", "",
         "One launch per kernel, `bench.py --profile-run` (eager, one view), clocks not locked "
         "(`--clock-control none`).  Units as ncu reports them.  Regenerate: `tools/r02_refresh_ncu.sh` "
         "on the GPU box, then this script.", ""]
traffic = {}
for key, rep in reports:
    raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                         capture_output=True, text=True).stdout.splitlines()))
    if len(raw) < 3:
        print("no data in", rep)
        continue
    h, units = raw[0], raw[1]
    col = {n: h.index(n) for n in h}
    lines += [f"## {WORKLOAD.get(key, key)} — `{os.path.basename(rep)}`", "",
              "| kernel | " + " | ".join(w[1] for w in WANT) + " |", "|---|" + "---|" * len(WANT)]
    seen = set()
    tr = traffic.setdefault(key, {})
    for row in raw[2:]:
        name = row[col["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "").split("<")[0].replace("inpc::", "")
        full = name.split("(")[0].replace("void ", "")
        if full in seen:
            continue
        seen.add(full)
        vals = [f"{row[col[m]]} {units[col[m]]}".strip() for m, _ in WANT]
        lines.append(f"| `{full}` | " + " | ".join(vals) + " |")
        st = STAGE.get(short)
        if st:
            def nbytes(m):
                v, u = float(row[col[m]]), units[col[m]]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            tr[st] = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
    lines.append("")
open(os.path.join(out_dir, f"{tag}_kernels.md"), "w").write("\n".join(lines) + "\n")
shutil.copy(launches, os.path.join(out_dir, f"{tag}_launches.csv"))
traffic["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes), one ncu --set full "
                   "capture per config; keys are bench.py's config/variant")
json.dump(traffic, open(os.path.join(out_dir, f"traffic_{tag}.json"), "w"), indent=1)
print("\n".join(lines))
print(json.dumps(traffic, indent=1))
