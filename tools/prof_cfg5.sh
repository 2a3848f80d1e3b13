mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_sort_big|k_blend_bwd" -s 200 -c 2 -o gpurun_out/prof_cfg5 python bench.py --config 5 --steps 1 --warmup 3 --profile-run --no-graph > gpurun_out/ncu_cfg5.log 2>&1
tail -3 gpurun_out/ncu_cfg5.log
