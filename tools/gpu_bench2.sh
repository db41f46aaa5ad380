set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c5w.json 2> gpurun_out/bench_c5w.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/bench_c5w_n2.json 2> gpurun_out/bench_c5w_n2.err
