mkdir -p gpurun_out
set -x
python bench.py > gpurun_out/bench_r01_a.json 2> gpurun_out/bench_r01_a.err
tail -c 3000 gpurun_out/bench_r01_a.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --profile-run > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_blend -s 8 -c 2 -o gpurun_out/prof_blend_r01 python bench.py --steps 3 --warmup 3 --profile-run > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_project|k_scan|k_sort" -s 8 -c 4 -o gpurun_out/prof_other_r01 python bench.py --steps 3 --warmup 3 --profile-run > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out
