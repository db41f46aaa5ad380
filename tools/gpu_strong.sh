set -x
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/mem.txt
timeout 900 python bench.py --config c5s --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/strong_n1.json 2> gpurun_out/strong_n1.err
for n in 2 4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2966$n bench.py --config c5s --gpus $n --steps 20 --warmup 3 --no-e2e > gpurun_out/strong_n$n.json 2> gpurun_out/strong_n$n.err; done
