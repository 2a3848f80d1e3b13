mkdir -p gpurun_out
for r in 1 2 3; do python bench.py --no-cpu-baseline --steps 300 > gpurun_out/bench_var$r.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_var$r.json')); print($r, round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, d['clocks'])"; done
python bench.py --no-cpu-baseline --config 5 --steps 5 --warmup 3 > gpurun_out/bench_cfg5b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_cfg5b.json')); print('cfg5', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()})"
