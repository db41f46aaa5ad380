set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 900 python tools/c3_node_level.py --ops srt27,cum27,cum19,srt19aa,cum19aa --scen A --vars V0,V1,V3 > gpurun_out/c3A.log 2>&1
rm -f gpurun_out/bench_next.jsonl
for c in c5w c5wpap c5wcum c5w64; do
  timeout 300 python bench.py --config $c --extra none --steps 20 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/$c /" >> gpurun_out/bench_next.jsonl 2>> gpurun_out/bench_next.err
done
