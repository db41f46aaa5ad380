set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "voxel" > gpurun_out/gputests_vox.log 2>&1; echo rc=$? >> gpurun_out/gputests_vox.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
