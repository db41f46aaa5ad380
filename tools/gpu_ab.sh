set -x
for c in c5wcum c4trt; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_b4.json 2> gpurun_out/bench_${c}_b4.err; done
