# weak scaling of the paper's configuration (c5wpap: D3Q19 cumulant AA fp64 + rotor pair per
# GPU; AA across ranks uses the NCCL ghost-plane copies) on N GPUs of one box
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python bench.py --config c5wpap --extra none --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/pap_n1.json 2> gpurun_out/pap_n1.err
for n in 2 4 8; do
  [ $n -le $N ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n bench.py --config c5wpap --extra none --gpus $n --steps 20 --warmup 5 > gpurun_out/pap_n$n.json 2> gpurun_out/pap_n$n.err
done
