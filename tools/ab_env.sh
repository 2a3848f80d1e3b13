#!/bin/bash
# A/B of env-var knobs on one bench config: ENVS="A=1 B=2;A=0" CFG=5 ARGS="--order morton"
mkdir -p gpurun_out
IFS=';' read -ra SETS <<< "$ENVS"
for e in "${SETS[@]}"; do
  env $e timeout 900 python bench.py --config ${CFG:-5} --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline $ARGS > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$e |', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()})" || tail -3 gpurun_out/ab.err
done
