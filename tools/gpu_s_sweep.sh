set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
for s in 0 1 2 3; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --s $s > gpurun_out/bench_s$s.json 2> gpurun_out/bench_s$s.err; done
