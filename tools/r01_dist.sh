mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "bands_assemble" 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config 4 --steps 5 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/bench_c4_2rank.json 2> gpurun_out/dist.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config 5 --steps 2 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/bench_c5_2rank.json 2>> gpurun_out/dist.err
tail -3 gpurun_out/dist.err
for f in c4_2rank c5_2rank; do head -c 900 gpurun_out/bench_$f.json; echo; done
