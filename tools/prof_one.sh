#!/bin/bash
# usage: tools/prof_one.sh CONFIG KERNEL_REGEX TAG [SKIP] [EXTRA_BENCH_ARGS]
# one ncu --set full capture of one kernel launch of bench.py --config CONFIG -> gpurun_out/prof_TAG.ncu-rep
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${4:-3} -c 1 -o gpurun_out/prof_$3 \
    python bench.py --config $1 --steps 1 --warmup 3 --profile-run --no-graph --no-cpu-baseline $5 > gpurun_out/ncu_$3.log 2>&1
tail -2 gpurun_out/ncu_$3.log
