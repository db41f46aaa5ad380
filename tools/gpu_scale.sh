# Multi-GPU check on N GPUs of one box (gpurun --gpus N --timeout 3000 -- 'bash tools/gpu_scale.sh'):
# bitwise multi-rank tests (fused and NCCL halo), weak (c5w) and strong (c5s) scaling, smoke.
set -x
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/gputests_mg.log 2>&1; echo rc=$? >> gpurun_out/gputests_mg.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/scale_n1.json 2> gpurun_out/scale_n1.err
timeout 600 python bench.py --config c5s --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/strong_n1.json 2> gpurun_out/strong_n1.err
for n in 2 4 8; do
  [ $n -le $N ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 50 --warmup 5 > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n bench.py --config c5s --gpus $n --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/strong_n$n.json 2> gpurun_out/strong_n$n.err
done
