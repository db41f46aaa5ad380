# Round-2 check on one B200: GPU tests, smoke, default bench (c5w64 + fp32 extra), Table I
# protocol, and the ncu evidence of the new default workload.
#   gpurun --timeout 3000 -- 'bash tools/gpu_r02a.sh'
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python tools/table1_cube.py --out gpurun_out/r02_table1_cube.md > gpurun_out/table1.log 2>&1
B="python bench.py --config c5w64 --extra none --steps 4 --warmup 3 --reps 1 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/plain_c5w64.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 5 -c 1 -o gpurun_out/prof_c5w64 $B > gpurun_out/ncu_c5w64.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5w64.csv $B > gpurun_out/ncu_launch64.log 2>&1
