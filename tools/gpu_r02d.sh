set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 600 python tools/kernel_sweep.py --only srt19f64,srt19f64aa,cum19f64,cum19f64aa,srt19f32,srt19f32aa,cum19f32aa,trt19f32aa,cum27f32,cum27f32aa,srt27f32aa,srt27f64aa,cum27f64aa > gpurun_out/sweep.log 2>&1
timeout 1800 python tools/settling_sphere.py --out gpurun_out/r02_settling_sphere.md > gpurun_out/settling.log 2>&1
