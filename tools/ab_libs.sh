# A/B: the in-tree lib (B) vs libinpc_raster_head.so (A): C<=4 parity tests on B, bench, optional ncu of one kernel ($K)
L=paper_2508_19140_b200/libinpc_raster.so
cp $L /tmp/new.so
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not channel_counts and not sh_features" 2>&1 | tail -2
for v in A B A B; do
  if [ $v = A ]; then cp paper_2508_19140_b200/libinpc_raster_head.so $L; else cp /tmp/new.so $L; fi
  timeout 600 python bench.py --config ${CFG:-2} --no-cpu-baseline --steps ${STEPS:-100} 2>/dev/null | tail -1 > gpurun_out/ab.json
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$v', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()})"
done
if [ -n "$K" ]; then
for v in A B; do
  if [ $v = A ]; then cp paper_2508_19140_b200/libinpc_raster_head.so $L; else cp /tmp/new.so $L; fi
  bash tools/ncu_quick.sh $K $v | grep -v "occupancy_limit\|registers_per"
done
fi
cp /tmp/new.so $L
