# The GPU parity suite against a library built with device-side bounds asserts
# (PSM_NVCC_EXTRA=-DPSM_BOUNDS_CHECK; build it here before the call, the .so travels with it).
set -x
export PSM_NVCC_EXTRA=-DPSM_BOUNDS_CHECK  # the stamp check in _build.py keeps this build
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seam.py tests/test_gpu_fullsize.py -x -q > gpurun_out/gputests_bounds.log 2>&1; echo rc=$? >> gpurun_out/gputests_bounds.log
