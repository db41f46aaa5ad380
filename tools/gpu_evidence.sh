# Round evidence batch on one B200 (gpurun --timeout 5000 -- 'bash tools/gpu_evidence.sh'):
# GPU tests, smoke, the default bench line (c5w64 + f32 + paper_config), the fluid-only
# collide sweep, the c3 node-level tables (R1 and R2), the s sweep, every NEXT-row workload,
# ncu of three collides and of the s = 2 mesh band pass
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python tools/kernel_sweep.py --only srt19f32,srt19f32aa,trt19f32,trt19f32aa,cum19f32,cum19f32aa,srt19f64,srt19f64aa,trt19f64,cum19f64,cum19f64aa,srt27f32,srt27f32aa,cum27f32,cum27f32aa,srt27f64,srt27f64aa,cum27f64,cum27f64aa > gpurun_out/sweep_all.log 2>&1
timeout 1800 python tools/c3_node_level.py --out gpurun_out/r02_c3_node_level.md --json gpurun_out/r02_c3_node_level.json > gpurun_out/c3.log 2>&1
timeout 900 python tools/c3_node_level.py --ops cum19aa,cum27 --mapping R2 --out gpurun_out/r02_c3_node_level_r2.md --json gpurun_out/r02_c3_node_level_r2.json > gpurun_out/c3r2.log 2>&1
bash tools/gpu_ssweep.sh
rm -f gpurun_out/bench_next.jsonl
for c in c5wpap c5wcum c5w27 c5wr2 c5app c4 c4aa c4f64 c4trt c4dyn c3f64 c3cum; do
  timeout 300 python bench.py --config $c --extra none --steps 20 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/$c /" >> gpurun_out/bench_next.jsonl 2>> gpurun_out/bench_next.err
done
for c in c5w64 c5wpap c5wcum; do
  B="python bench.py --config $c --extra none --steps 4 --warmup 3 --reps 1 --no-cpu-baseline --no-e2e"
  timeout 300 $B > gpurun_out/plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 5 -c 2 -o gpurun_out/prof_$c $B > gpurun_out/ncu_$c.log 2>&1
done
B="python bench.py --config c5w64 --extra none --steps 4 --warmup 3 --reps 1 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5w64.csv $B > gpurun_out/ncu_launch64.log 2>&1
B="python tools/c3_node_level.py --ops cum19aa --scen A --vars V4 --steps 4 --warmup 1 --reps 1"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_remap_l3_mesh -s 8 -c 1 -o gpurun_out/prof_remap_l3_mesh $B > gpurun_out/ncu_remap.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3A_V4.csv $B > /dev/null 2>&1
