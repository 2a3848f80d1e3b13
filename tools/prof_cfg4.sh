mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_sort_big" -s 3 -c 1 -o gpurun_out/prof_cfg4 python bench.py --config 4 --steps 1 --warmup 3 --profile-run --no-graph > gpurun_out/ncu_cfg4.log 2>&1
tail -2 gpurun_out/ncu_cfg4.log
