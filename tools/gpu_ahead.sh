set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
for b in 1184 296 148 64 32 16; do PSM_AHEAD_BLOCKS=$b timeout 300 python bench.py --config c5w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5w_b$b.json 2> gpurun_out/bench_c5w_b$b.err; done
PSM_NO_REMAP_AHEAD=1 timeout 300 python bench.py --config c5w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5w_noahead.json 2> gpurun_out/bench_c5w_noahead.err
