#!/bin/bash
# quick GPU check: parity suite + cfg2 bench stage times (+ optional extra configs in $CFGS)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 2 ${CFGS}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/quick_cfg$c.json
  python -c "import json; d=json.load(open('gpurun_out/quick_cfg$c.json')); print($c, round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done
for v in ${VARIANTS}; do
  timeout 600 python bench.py --variant $v --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/quick_$v.json
  python -c "import json; d=json.load(open('gpurun_out/quick_$v.json')); print('$v', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done
