set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k degenerate > gpurun_out/gputests_deg.log 2>&1; echo rc=$? >> gpurun_out/gputests_deg.log
