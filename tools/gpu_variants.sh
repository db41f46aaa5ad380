# kernel-tuning experiment: the collide sweep (and optionally the c3 scenario-A static PSM run)
# with every variant library under paper_2502_20049_b200/variants/ (built here with
# _build.build(out=..., extra_flags=...)), alternated twice to separate library effects from
# box drift
mkdir -p gpurun_out
ONLY=${ONLY:-srt19f64aa,cum19f64aa,srt19f32aa,cum19f32aa,srt19f64}
for round in 1 2; do
for v in paper_2502_20049_b200/variants/*.so; do
  echo "== $v" >> gpurun_out/variants.log
  PSM_LIB=$v timeout 300 python tools/kernel_sweep.py --only $ONLY $SWEEP_ARGS >> gpurun_out/variants.log 2>&1
  if [ -n "$C3OPS" ]; then
    PSM_LIB=$v timeout 600 python tools/c3_node_level.py --ops $C3OPS --scen A --vars V1 --steps 20 --reps 3 2>&1 | grep "^{" >> gpurun_out/variants.log
  fi
done
done
cat gpurun_out/variants.log
