#!/bin/bash
# ncu --set full of one launch each of the cfg5 kernels; summaries on the box, big reports dropped
mkdir -p gpurun_out
T=${1:-c5}; shift
KS=${KS:-"k_sort_big k_blend_fwd k_blend_bwd k_project_count k_scatter_slots"}
for k in $KS; do
ncu --set full --clock-control none --import-source on -k regex:"$k" -s 70 -c 1 -o gpurun_out/prof_${T}_$k \
    python bench.py --config 5 --steps 1 --warmup 3 --profile-run --no-graph --no-cpu-baseline "$@" > gpurun_out/ncu_${T}_$k.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_${T}_$k.ncu-rep 25 > gpurun_out/sum_${T}_$k.txt 2>&1
python tools/stall_regions.py gpurun_out/prof_${T}_$k.ncu-rep $k 60 >> gpurun_out/sum_${T}_$k.txt 2>&1
sz=$(stat -c %s gpurun_out/prof_${T}_$k.ncu-rep 2>/dev/null || echo 0)
if [ "$sz" -gt 12000000 ]; then rm -f gpurun_out/prof_${T}_$k.ncu-rep; fi
done
du -sh gpurun_out
