set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
for v in "c5w 1 0" "c5w 0 0" "c5wr2 1 0" "c4 1 0" "c5w 1 1" "c5w 0 1" "c5wcum 1 0"; do set -- $v; if [ $3 = 1 ]; then export PSM_NO_REMAP_AHEAD=1; else unset PSM_NO_REMAP_AHEAD; fi; PSM_BAND_CACHE=$2 timeout 300 python bench.py --config $1 --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/$1_cache$2_noahead$3 /" >> gpurun_out/bench_rep.jsonl 2>> gpurun_out/bench_rep.err; done
