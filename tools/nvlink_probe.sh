# which NVLink traffic counters this box exposes (run on >= 2 GPUs)
mkdir -p gpurun_out
{ nvidia-smi nvlink -s -i 0 | head -8; nvidia-smi nvlink -gt d -i 0 | head -8; nvidia-smi nvlink -h | grep -i -A2 "throughput\|counter" | head -30; } > gpurun_out/nvlink_probe.txt 2>&1
python - >> gpurun_out/nvlink_probe.txt 2>&1 <<'PY'
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
for f in ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX"):
    fid = getattr(nv, f)
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(f, scope, v.nvmlReturn, v.valueType, v.value.ullVal)
        except Exception as e:
            print(f, scope, "exc", e)
for link in range(2):
    try:
        print("util ctr", link, nv.nvmlDeviceGetNvLinkUtilizationCounter(h, link, 0))
    except Exception as e:
        print("util ctr exc", e)
    try:
        print("state", link, nv.nvmlDeviceGetNvLinkState(h, link))
    except Exception as e:
        print("state exc", e)
PY
# counters around a 2-rank fused-halo run of the default workload (fp64 c5w64, 40 steps)
nvidia-smi nvlink -gt d > gpurun_out/nvlink_before.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 2 --steps 40 --warmup 3 --reps 1 --extra none --no-e2e > gpurun_out/nvlink_bench.json 2> gpurun_out/nvlink_bench.err
nvidia-smi nvlink -gt d > gpurun_out/nvlink_after.txt 2>&1
