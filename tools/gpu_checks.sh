# correctness check of the final code: the GPU parity, seam and full-size suites against the
# bounds-asserting build (PSM_LIB=variants/bounds.so, built here before the call with
# _build.build(out=..., extra_flags="-DPSM_BOUNDS_CHECK"); compute-sanitizer is closed on the pool)
mkdir -p gpurun_out
PSM_LIB=paper_2502_20049_b200/variants/bounds.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seam.py tests/test_gpu_fullsize.py -x -q > gpurun_out/gputests_bounds.log 2>&1; echo rc=$? >> gpurun_out/gputests_bounds.log
