set -x
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/gputests_mg.log 2>&1; echo rc=$? >> gpurun_out/gputests_mg.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --steps 40 --warmup 4 --no-e2e > gpurun_out/scale_n2.json 2> gpurun_out/scale_n2.err
