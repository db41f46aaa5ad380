set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
for c in c5w c4 c5wr2; do timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
PSM_BAND_CACHE=0 timeout 300 python bench.py --config c5w --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5w_nocache.json 2> gpurun_out/bench_c5w_nocache.err
PSM_NO_REMAP_AHEAD=1 timeout 300 python bench.py --config c5w --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5w_noahead.json 2> gpurun_out/bench_c5w_noahead.err
