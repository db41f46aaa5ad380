set -x
rm -f gpurun_out/bench_abl.jsonl
for c in c5w27 c5wcum; do timeout 300 python bench.py --config $c --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/$c /" >> gpurun_out/bench_abl.jsonl 2>> gpurun_out/bench_abl.err; done
