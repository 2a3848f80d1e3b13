#!/bin/bash
# round-2 start: parity suite + headline bench + cfg5 bench + launch list (one GPU)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_gpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu.log 2>&1; tail -3 gpurun_out/r02_pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02_base_cfg2.json 2> gpurun_out/r02_base_cfg2.err
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_base_cfg5.json 2> gpurun_out/r02_base_cfg5.err
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/r02_base_cfg4.json 2> gpurun_out/r02_base_cfg4.err
for f in gpurun_out/r02_base_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, d['roofline']['kernel'], round(d['roofline']['frac'],3))"; done
