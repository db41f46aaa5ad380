set -x
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/scale_n1.json 2> gpurun_out/scale_n1.err
for n in 2 4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 50 --warmup 5 > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err; done
timeout 900 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/gputests_mg.log 2>&1; echo rc=$? >> gpurun_out/gputests_mg.log
