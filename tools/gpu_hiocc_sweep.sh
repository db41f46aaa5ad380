# fp64 D3Q19 occupancy variants fluid-only (kernel sweep) per operator/pattern: PSM_HIOCC=0/1
mkdir -p gpurun_out
for r in 1 2; do for h in 0 1; do
  echo "== hiocc$h" >> gpurun_out/hiocc_sweep.log
  PSM_HIOCC=$h timeout 600 python tools/kernel_sweep.py --only srt19f64,srt19f64aa,trt19f64,cum19f64,cum19f64aa >> gpurun_out/hiocc_sweep.log 2>&1
done; done
