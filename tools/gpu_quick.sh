set -x
rm -f gpurun_out/bench_abl.jsonl
for rep in 1 2; do for pr in high low; do PSM_AHEAD_PRIO=$pr timeout 300 python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/c5w-$pr /" >> gpurun_out/bench_abl.jsonl 2>> gpurun_out/bench_abl.err; done; done
