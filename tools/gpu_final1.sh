set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in c5app c5wr2 c4 c4aa c4f64 c4trt c4dyn c3f64 c3cum c5wcum; do timeout 300 python bench.py --config $c --steps 40 --warmup 3 --no-cpu-baseline | sed "s/^/$c /" >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err; done
PSM_NO_REMAP_AHEAD=1 timeout 300 python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/c5w-noahead /" >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 5 -c 1 -o gpurun_out/prof_c5w_final2 $B > gpurun_out/ncu_c5w.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5w.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
