#!/bin/bash
# GPU check of a diagnostics build (-DINPC_FAST_BUILD: C <= 4 kernels only):
# the C <= 4 parity tests + the cfg2 bench line (stage times, roofline)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not channel_counts and not sh_features" ${PYTEST_EXTRA} 2>&1 | tail -3
for c in 2 ${CFGS}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline 2>gpurun_out/fc_err$c.txt | tail -1 > gpurun_out/fc_cfg$c.json
  python -c "import json; d=json.load(open('gpurun_out/fc_cfg$c.json')); print($c, round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, d['roofline']['kernel'], round(d['roofline']['frac'],3))" || tail -5 gpurun_out/fc_err$c.txt
done
