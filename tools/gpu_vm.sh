set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "two_way" > gpurun_out/gputests_vm.log 2>&1; echo rc=$? >> gpurun_out/gputests_vm.log
timeout 1200 python tools/settling_sphere.py --out gpurun_out/settling.md > gpurun_out/settling.log 2>&1
