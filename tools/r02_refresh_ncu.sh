#!/bin/bash
# ncu evidence for profiles/ (one GPU, round 2): launch list of the default bench step (cfg5, 64 views),
# one --set full launch of each cfg5 kernel, cfg2 kernels, the dominant kernel of cfg3 / cfg4 / variants
mkdir -p gpurun_out/prof_out
B="python bench.py --steps 1 --warmup 3 --profile-run --no-graph --no-cpu-baseline"
# launch list: skip the stats forward (64 x 7 kernels) + 3 warm-up steps of 64 views (8 kernels per view), keep one step
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -s 1984 -c 512 --csv \
    --log-file gpurun_out/launches_r02.csv $B > /dev/null 2>&1
for k in k_blend_bwd k_blend_fwd k_sort_mid k_project_count k_scatter_slots k_scan_tiles; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s 70 -c 1 -o gpurun_out/prof_r02_cfg5_$k $B > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_(bin|blend)" -s 6 -c 3 \
    -o gpurun_out/prof_r02_cfg2 $B --config 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_blend_fwd" -s 2 -c 1 -o gpurun_out/prof_r02_cfg3 $B --config 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_sort_big" -s 2 -c 1 -o gpurun_out/prof_r02_cfg4 $B --config 4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_blend_bwd" -s 2 -c 1 -o gpurun_out/prof_r02_env $B --config 2 --variant env > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_blend_bwd" -s 2 -c 1 -o gpurun_out/prof_r02_sh $B --config 2 --variant sh > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
PROFILE_OUT=gpurun_out/prof_out python tools/make_profile_summary.py r02 gpurun_out/launches_r02.csv \
    cfg5=gpurun_out/prof_r02_cfg5_k_blend_bwd.ncu-rep cfg5=gpurun_out/prof_r02_cfg5_k_blend_fwd.ncu-rep \
    cfg5=gpurun_out/prof_r02_cfg5_k_sort_mid.ncu-rep cfg5=gpurun_out/prof_r02_cfg5_k_project_count.ncu-rep \
    cfg5=gpurun_out/prof_r02_cfg5_k_scatter_slots.ncu-rep cfg5=gpurun_out/prof_r02_cfg5_k_scan_tiles.ncu-rep \
    cfg2=gpurun_out/prof_r02_cfg2.ncu-rep cfg3=gpurun_out/prof_r02_cfg3.ncu-rep \
    cfg4=gpurun_out/prof_r02_cfg4.ncu-rep cfg2-env=gpurun_out/prof_r02_env.ncu-rep \
    cfg2-sh=gpurun_out/prof_r02_sh.ncu-rep > gpurun_out/prof_out/summary.log 2>&1
for k in cfg5_k_blend_bwd cfg5_k_blend_fwd cfg5_k_sort_mid cfg5_k_project_count; do
  python tools/stall_regions.py gpurun_out/prof_r02_$k.ncu-rep ${k#cfg5_} 4000 > gpurun_out/prof_out/stall_$k.txt 2>&1
done
for k in k_bin k_blend_bwd k_blend_fwd; do
  python tools/stall_regions.py gpurun_out/prof_r02_cfg2.ncu-rep $k 4000 > gpurun_out/prof_out/stall_cfg2_$k.txt 2>&1
done
mkdir -p /tmp/ncu_reps && mv gpurun_out/*.ncu-rep /tmp/ncu_reps/
ls gpurun_out/prof_out
