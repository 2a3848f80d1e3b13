mkdir -p gpurun_out
python bench.py --no-cpu-baseline --variant sh > gpurun_out/bench_sh.json 2> gpurun_out/bench_var.err
python bench.py --no-cpu-baseline --variant env > gpurun_out/bench_env.json 2>> gpurun_out/bench_var.err
python bench.py --no-cpu-baseline --config 5 --steps 5 --warmup 3 > gpurun_out/bench_cfg5.json 2>> gpurun_out/bench_var.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 20 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/bench_2rank_gloo.json 2>> gpurun_out/bench_var.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench_var.err
tail -5 gpurun_out/bench_var.err
for f in gpurun_out/bench_sh.json gpurun_out/bench_env.json gpurun_out/bench_cfg5.json gpurun_out/bench_2rank_gloo.json gpurun_out/bench_ref.json; do echo $f; head -c 600 $f; echo; done
