#!/bin/bash
# k_bin_bilinear phase times (diagnostic build with -DINPC_PHASE_TIMES [+ $EXTRA]; BENCH_ARGS e.g. "--config 5")
INPC_NVCC_EXTRA="-DINPC_PHASE_TIMES $EXTRA" python paper_2508_19140_b200/build.py --force > /dev/null 2>&1
python bench.py --no-cpu-baseline --no-graph --steps 3 --warmup 3 ${BENCH_ARGS} 2>&1 | grep "bin phases" | tail -3
