set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 1500 python tools/c3_node_level.py --out gpurun_out/r02_c3_node_level.md --json gpurun_out/r02_c3_node_level.json > gpurun_out/c3.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
rm -f gpurun_out/bench_next.jsonl
for c in c5wpap c5wcum c5w27 c4; do
  timeout 300 python bench.py --config $c --extra none --steps 20 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/$c /" >> gpurun_out/bench_next.jsonl 2>> gpurun_out/bench_next.err
done
