set -x
timeout 600 python tools/settling_sphere.py --out gpurun_out/settling.md > gpurun_out/settling.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
