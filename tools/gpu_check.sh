set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
for c in c4 c4aa c4f64 c3f64; do timeout 200 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 6 -c 1 -o gpurun_out/prof_c4b python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
