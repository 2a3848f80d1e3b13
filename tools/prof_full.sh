# usage: bash tools/prof_full.sh TAG  -> gpurun_out/prof_TAG.ncu-rep (one launch of each kernel)
mkdir -p gpurun_out
TAG=${1:-x}
ncu --set full --clock-control none --import-source on -k regex:"k_(project|scan|scatter|sort|blend|bin)" -s 6 -c 3 \
    -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --profile-run > gpurun_out/ncu_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 40 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --profile-run > /dev/null 2>&1
tail -3 gpurun_out/ncu_$TAG.log
