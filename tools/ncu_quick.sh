#!/bin/bash
# instruction count, duration, issue activity and top stall reasons of one launch of a kernel (cfg2 unless $CFG)
# usage: tools/ncu_quick.sh KERNEL_REGEX [TAG]
mkdir -p gpurun_out
ncu --clock-control none -k regex:"$1" -s 3 -c 1 \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio,smsp__average_warp_latency_issue_stalled_wait.ratio,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers \
  --csv --log-file gpurun_out/nq_${2:-x}.csv python bench.py --config ${CFG:-2} --steps 1 --warmup 3 --profile-run --no-graph --no-cpu-baseline > /dev/null 2>&1
python - "$1" gpurun_out/nq_${2:-x}.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
for r in rows[1:]:
    print(r[ki][:40], r[mi], r[vi], r[ui])
PY
