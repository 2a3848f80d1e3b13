mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline --steps 300 > gpurun_out/bench_c2.json 2>gpurun_out/c34.err
python bench.py --no-cpu-baseline --config 3 --steps 50 > gpurun_out/bench_c3.json 2>>gpurun_out/c34.err
python bench.py --no-cpu-baseline --config 4 --steps 20 > gpurun_out/bench_c4.json 2>>gpurun_out/c34.err
tail -3 gpurun_out/c34.err
for f in c2 c3 c4; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, d['roofline']['kernel'], round(d['roofline']['frac'],3), d['cuda_graph'], d['config']['F_t'])"; done
python bench.py --no-cpu-baseline --config 5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2>>gpurun_out/c34.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c5.json')); print('c5', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, d['roofline']['kernel'], round(d['roofline']['frac'],3))"
