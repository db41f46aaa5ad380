set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cumulant or paper" > gpurun_out/cum_tests.log 2>&1; echo rc=$? >> gpurun_out/cum_tests.log
ONLY=cum27f32,cum19f32,cum19f32aa,cum27f32aa,cum19f64aa,cum27f64 bash tools/gpu_variants.sh > /dev/null 2>&1
