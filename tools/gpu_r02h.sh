mkdir -p gpurun_out
for n in 256 384 512; do
  timeout 900 python tools/kernel_sweep.py --n $n --only cum19f64aa,srt19f64aa,cum19f64,srt19f64 --pads 0,288,4128 --reps 5 >> gpurun_out/pad.log 2>&1
done
