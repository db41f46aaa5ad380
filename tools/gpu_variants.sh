# kernel-tuning experiment: the collide sweep with every variant library under
# paper_2502_20049_b200/variants/ (built here with _build.build(out=..., extra_flags=...)),
# alternated twice to separate library effects from box drift
mkdir -p gpurun_out
ONLY=${ONLY:-srt19f64aa,cum19f64aa,srt19f32aa,cum19f32aa,srt19f64}
for round in 1 2; do
for v in paper_2502_20049_b200/variants/*.so; do
  echo "== $v" >> gpurun_out/variants.log
  PSM_LIB=$v timeout 300 python tools/kernel_sweep.py --only $ONLY $SWEEP_ARGS >> gpurun_out/variants.log 2>&1
done
done
cat gpurun_out/variants.log
