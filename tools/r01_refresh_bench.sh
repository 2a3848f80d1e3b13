#!/bin/bash
# the bench lines committed under profiles/ (one GPU): headline (with the CPU oracle baseline),
# the reference arm, the NEXT-row variants, configs 3/4/5, the f4 sort A/B, 2-rank gloo runs on one GPU
mkdir -p gpurun_out
B=gpurun_out/final
python bench.py > ${B}_bench.json 2> ${B}_bench.err
python bench.py --impl reference > ${B}_reference.json 2>> ${B}_bench.err
python bench.py --variant sh --no-cpu-baseline > ${B}_sh.json 2>> ${B}_bench.err
python bench.py --variant env --no-cpu-baseline > ${B}_env.json 2>> ${B}_bench.err
python bench.py --config 3 --no-cpu-baseline > ${B}_cfg3.json 2>> ${B}_bench.err
python bench.py --config 4 --no-cpu-baseline > ${B}_cfg4.json 2>> ${B}_bench.err
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > ${B}_cfg5.json 2>> ${B}_bench.err
python bench.py --sort-ab > ${B}_sort_ab.json 2>> ${B}_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --dist-backend gloo --no-cpu-baseline > ${B}_2rank_gloo.json 2>> ${B}_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
    bench.py --gpus 2 --config 4 --dist-backend gloo --no-cpu-baseline > ${B}_cfg4_2rank_gloo.json 2>> ${B}_bench.err
tail -3 ${B}_bench.err
for f in ${B}_*.json; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1])
except Exception as e:
    print('$f', 'unparsable', e); sys.exit()
print('$f', d.get('value'), d.get('unit'), d.get('ms_per_step'), (d.get('roofline') or {}).get('kernel'), round((d.get('roofline') or {}).get('frac', 0) or 0, 3))"; done
