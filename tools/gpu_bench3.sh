set -x
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e > gpurun_out/bench_c5w_n2.json 2> gpurun_out/bench_c5w_n2.err
