mkdir -p gpurun_out
python bench.py --no-cpu-baseline --steps 300 > gpurun_out/bench_a.json 2>/dev/null
INPC_FUSED_BIN_IN_GRAPH=1 python bench.py --no-cpu-baseline --steps 300 > gpurun_out/bench_b.json 2>/dev/null
for f in a b; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()})"; done
