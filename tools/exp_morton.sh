#!/bin/bash
mkdir -p gpurun_out
for o in given morton; do
for c in 5 4; do
timeout 600 python bench.py --config $c --order $o --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/exp_${o}_cfg$c.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/exp_${o}_cfg$c.json').read().strip().splitlines()[-1])
print('$o $c', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done; done
