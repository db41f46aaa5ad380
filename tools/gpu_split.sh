# overlapped remap (collide of the untouched tile columns during the remap): all GPU tests, the
# fluid-only sweep (code generation check), then split on/off for the default line with its e2e,
# c5w at s = 3 (remap in series) and c3 scenario A V4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/split_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/split_tests.log
timeout 900 python tools/kernel_sweep.py --only srt19f32,srt19f32aa,cum19f32aa,cum27f32aa,cum27f32,srt19f64,srt19f64aa,cum19f64aa,cum27f64aa > gpurun_out/split_sweep.log 2>&1
for r in 1 2; do for f in 0 1; do
  if [ $f = 0 ]; then export PSM_NO_SPLIT=1; else unset PSM_NO_SPLIT; fi
  echo "== split$f" >> gpurun_out/split.log
  timeout 400 python bench.py --extra none --steps 20 --warmup 3 --reps 3 --no-cpu-baseline >> gpurun_out/split.log 2>&1
  timeout 300 python bench.py --config c5w --extra none --s 3 --steps 20 --warmup 3 --reps 3 --no-cpu-baseline --no-e2e >> gpurun_out/split.log 2>&1
  timeout 300 python tools/c3_node_level.py --ops cum19aa --scen A --vars V4 --steps 20 --reps 3 2>&1 | grep "^{" >> gpurun_out/split.log
done; done
unset PSM_NO_SPLIT
