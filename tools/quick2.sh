#!/bin/bash
# parity suite + bench lines of $CFGS (default 5 4) -> one-line summaries
mkdir -p gpurun_out
T=${TAG:-q}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log
for c in ${CFGS:-5 4}; do
st=3; [ $c = 5 ] || st=20
timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline ${BENCH_EXTRA} > gpurun_out/${T}_cfg$c.json 2>gpurun_out/${T}_cfg$c.err
python -c "
import json
d=json.loads(open('gpurun_out/${T}_cfg$c.json').read().strip().splitlines()[-1])
print('$c', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, d['roofline']['kernel'], round(d['roofline']['frac'],3))" || tail -3 gpurun_out/${T}_cfg$c.err
done
