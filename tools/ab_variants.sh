#!/bin/bash
# A/B of variant libraries (tools/build_variant.sh) on the cfg $CFG bench: VARIANTS="base f8 ..."
L=paper_2508_19140_b200/libinpc_raster.so
cp $L /tmp/orig.so
mkdir -p gpurun_out
for r in 1 2; do
for v in $VARIANTS; do
  cp paper_2508_19140_b200/libinpc_raster_$v.so $L
  timeout 600 python bench.py --config ${CFG:-5} --no-cpu-baseline --steps ${STEPS:-10} --warmup 3 2>/dev/null | tail -1 > gpurun_out/ab_$v.json
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['value'],1), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms_per_step'].items()})"
done
done
cp /tmp/orig.so $L
