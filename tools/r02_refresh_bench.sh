#!/bin/bash
# the bench lines committed under profiles/ (one GPU, round 2)
mkdir -p gpurun_out
B=gpurun_out/r02
python bench.py > ${B}_bench.json 2> ${B}_bench.err
python bench.py --impl reference > ${B}_reference.json 2>> ${B}_bench.err
python bench.py --config 2 --steps 200 --warmup 10 > ${B}_cfg2.json 2>> ${B}_bench.err
python bench.py --config 2 --variant sh --steps 100 --no-cpu-baseline > ${B}_sh.json 2>> ${B}_bench.err
python bench.py --config 2 --variant env --steps 100 --no-cpu-baseline > ${B}_env.json 2>> ${B}_bench.err
python bench.py --config 3 --steps 100 --no-cpu-baseline > ${B}_cfg3.json 2>> ${B}_bench.err
python bench.py --config 4 --steps 50 --no-cpu-baseline > ${B}_cfg4.json 2>> ${B}_bench.err
python bench.py --sort-ab > ${B}_sort_ab.json 2>> ${B}_bench.err
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 5 --no-cpu-baseline > ${B}_2rank_gloo.json 2>> ${B}_bench.err
timeout 900 python bench.py --gpus 2 --config 4 --dist-backend gloo --steps 10 --no-cpu-baseline > ${B}_cfg4_2rank_gloo.json 2>> ${B}_bench.err
tail -3 ${B}_bench.err
for f in ${B}_*.json; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1])
except Exception as e:
    print('$f', 'unparsable', e); sys.exit()
print('$f', d.get('value'), d.get('unit'), d.get('ms_per_step'), (d.get('roofline') or {}).get('kernel'), round((d.get('roofline') or {}).get('frac', 0) or 0, 3), (d.get('step_roofline') or {}).get('frac'))"; done
