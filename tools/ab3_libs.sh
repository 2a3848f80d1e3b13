#!/bin/bash
# three-way: head (A), mid (M), in-tree (B); bench stage times for $CFG
L=paper_2508_19140_b200/libinpc_raster.so
cp $L /tmp/new.so
for v in A M B A M B; do
  case $v in A) cp paper_2508_19140_b200/libinpc_raster_head.so $L;; M) cp paper_2508_19140_b200/libinpc_raster_mid.so $L;; B) cp /tmp/new.so $L;; esac
  timeout 600 python bench.py --config ${CFG:-2} --no-cpu-baseline --steps ${STEPS:-100} 2>/dev/null | tail -1 > gpurun_out/ab.json
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$v', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()})"
done
cp /tmp/new.so $L
