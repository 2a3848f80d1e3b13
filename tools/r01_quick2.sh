mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python bench.py --no-cpu-baseline --variant sh > gpurun_out/bench_${TAG}_sh.json 2>> gpurun_out/bench_$TAG.err
python bench.py --no-cpu-baseline --variant env > gpurun_out/bench_${TAG}_env.json 2>> gpurun_out/bench_$TAG.err
python bench.py --no-cpu-baseline --config 5 --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_cfg5.json 2>> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err
for f in gpurun_out/bench_$TAG.json gpurun_out/bench_${TAG}_sh.json gpurun_out/bench_${TAG}_env.json gpurun_out/bench_${TAG}_cfg5.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],1), 'fps', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, 'frac', round(d['step_roofline']['frac'],3))"; done
