# D3Q19 cumulant parity + the paper-configuration bench + the c3 node-level experiment
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cumulant or paper" > gpurun_out/cum_tests.log 2>&1; echo rc=$? >> gpurun_out/cum_tests.log
timeout 600 python bench.py --config c5wpap --extra none --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5wpap.json 2> gpurun_out/bench_c5wpap.err
timeout 600 python bench.py --config c5wcum --extra none --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5wcum.json 2> gpurun_out/bench_c5wcum.err
timeout 1500 python tools/c3_node_level.py --out gpurun_out/r02_c3_node_level.md --json gpurun_out/r02_c3_node_level.json > gpurun_out/c3.log 2>&1
