set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cumulant" > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
rm -f gpurun_out/bench_abl.jsonl
for c in c5wcum c3cum; do timeout 300 python bench.py --config $c --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/$c /" >> gpurun_out/bench_abl.jsonl 2>> gpurun_out/bench_abl.err; done
