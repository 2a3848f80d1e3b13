#!/bin/bash
# ncu evidence for profiles/ (one GPU): cfg2 kernels + launch list, the dominant kernel of every other bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
ncu --set full --clock-control none --import-source on -k regex:"k_(bin|blend)" -s 6 -c 3 \
    -o gpurun_out/prof_final_cfg2 python bench.py --steps 3 --warmup 3 --profile-run --no-cpu-baseline > gpurun_out/ncu_final_cfg2.log 2>&1
tail -1 gpurun_out/ncu_final_cfg2.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 40 --csv \
    --log-file gpurun_out/launches_final.csv python bench.py --steps 3 --warmup 3 --profile-run --no-cpu-baseline > /dev/null 2>&1
tools/prof_one.sh 3 "k_blend_fwd" final_cfg3 2
tools/prof_one.sh 4 "k_sort_big" final_cfg4 2
tools/prof_one.sh 5 "k_blend_bwd" final_cfg5 2
tools/prof_one.sh 2 "k_blend_bwd" final_env 2 "--variant env"
tools/prof_one.sh 2 "k_blend_bwd" final_sh 2 "--variant sh"
ls -la gpurun_out/*.ncu-rep | tail -8
# summaries on the box (the reports together exceed what gpurun brings back)
PROFILE_OUT=gpurun_out/prof_out python tools/make_profile_summary.py r01 gpurun_out/launches_final.csv \
    cfg2=gpurun_out/prof_final_cfg2.ncu-rep cfg3=gpurun_out/prof_final_cfg3.ncu-rep \
    cfg4=gpurun_out/prof_final_cfg4.ncu-rep cfg5=gpurun_out/prof_final_cfg5.ncu-rep \
    cfg2-env=gpurun_out/prof_final_env.ncu-rep cfg2-sh=gpurun_out/prof_final_sh.ncu-rep > /dev/null
for k in cfg2:k_blend_bwd cfg2:k_blend_fwd cfg2:k_bin cfg3:k_blend_fwd cfg4:k_sort_big cfg5:k_blend_bwd; do
  python tools/src_lines.py gpurun_out/prof_final_${k%%:*}.ncu-rep ${k##*:} 40 > gpurun_out/prof_out/src_${k%%:*}_${k##*:}.txt 2>&1
  python tools/stall_regions.py gpurun_out/prof_final_${k%%:*}.ncu-rep ${k##*:} 4000 > gpurun_out/prof_out/stall_${k%%:*}_${k##*:}.txt 2>&1
done
mkdir -p /tmp/ncu_reps && mv gpurun_out/prof_final_cfg[345].ncu-rep gpurun_out/prof_final_env.ncu-rep gpurun_out/prof_final_sh.ncu-rep /tmp/ncu_reps/
ls gpurun_out/prof_out
