set -x
for c in c4aa c4 c5w; do timeout 300 python bench.py --config $c --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/$c /" >> gpurun_out/bench_abl.jsonl 2>> gpurun_out/bench_abl.err; done
