# Multi-GPU check on N GPUs of one box (gpurun --gpus N --timeout 3000 -- 'bash tools/gpu_scale.sh'):
# bitwise multi-rank tests (fused and NCCL halo, with and without bodies), weak scaling of the
# default line (c5w64 fp64 + the fp32 c5w beside it), strong scaling (c5s), and the application
# run with open boundaries (c5app), each with NVML NVLink counters around the timed steps.
set -x
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/gputests_mg.log 2>&1; echo rc=$? >> gpurun_out/gputests_mg.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/scale_n1.json 2> gpurun_out/scale_n1.err
timeout 600 python bench.py --config c5app --extra none --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/app_n1.json 2> gpurun_out/app_n1.err
timeout 600 python bench.py --config c5s --extra none --steps 10 --warmup 3 --reps 3 --no-cpu-baseline --no-e2e > gpurun_out/strong_n1.json 2> gpurun_out/strong_n1.err
for n in 2 4 8; do
  [ $n -le $N ] || continue
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  timeout 900 $R --master-port 2955$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err
  timeout 900 $R --master-port 2957$n bench.py --config c5app --extra none --gpus $n --steps 20 --warmup 5 > gpurun_out/app_n$n.json 2> gpurun_out/app_n$n.err
  PSM_HALO=nccl timeout 900 $R --master-port 2958$n bench.py --config c5app --extra none --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/app_nccl_n$n.json 2> gpurun_out/app_nccl_n$n.err
  timeout 900 $R --master-port 2956$n bench.py --config c5s --extra none --gpus $n --steps 10 --warmup 3 --reps 3 --no-cpu-baseline --no-e2e > gpurun_out/strong_n$n.json 2> gpurun_out/strong_n$n.err
done
