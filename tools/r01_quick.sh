# quick: gpu tests + bench (graph) + bench (eager)
mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python bench.py --no-cpu-baseline --no-graph > gpurun_out/bench_${TAG}_eager.json 2>> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err
for f in gpurun_out/bench_$TAG.json gpurun_out/bench_${TAG}_eager.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']), 'fps', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, 'frac', round(d['step_roofline']['frac'],3), 'graph', d.get('cuda_graph'), 'launches', d['gpu_launches'])"; done
