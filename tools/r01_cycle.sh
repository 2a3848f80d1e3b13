# test + bench + profile cycle: bash tools/r01_cycle.sh TAG
mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 1500 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
bash tools/prof_full.sh $TAG
