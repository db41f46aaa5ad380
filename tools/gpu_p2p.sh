set -x
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/gputests_mg.log 2>&1; echo rc=$? >> gpurun_out/gputests_mg.log
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus $N --steps 30 --warmup 5 --no-e2e > gpurun_out/p2p_n$N.json 2> gpurun_out/p2p_n$N.err
PSM_HALO=nccl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29553 bench.py --gpus $N --steps 30 --warmup 5 --no-e2e > gpurun_out/nccl_n$N.json 2> gpurun_out/nccl_n$N.err
