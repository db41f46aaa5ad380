set -x
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_c5w.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_map -s 4 -c 1 -o gpurun_out/prof_map python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_map.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -k cror -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
