# kernel-tuning experiment: the collide sweep with every variant library under
# paper_2502_20049_b200/variants/ (built here with _build.build(out=..., extra_flags=...)),
# plus ncu counters of the AA kernels of the base library and of $NCU_VARIANT
mkdir -p gpurun_out
ONLY=${ONLY:-srt19f64aa,cum19f64aa,srt19f32aa,cum19f32aa,srt19f64}
for v in paper_2502_20049_b200/variants/*.so; do
  echo "== $v" >> gpurun_out/variants.log
  PSM_LIB=$v timeout 300 python tools/kernel_sweep.py --only $ONLY >> gpurun_out/variants.log 2>&1
done
cat gpurun_out/variants.log
if [ -n "$NCU_ONLY" ]; then
  timeout 900 ncu --set full --clock-control none -k regex:k_collide -s 4 -c 4 -o gpurun_out/prof_sweep python tools/kernel_sweep.py --only $NCU_ONLY --steps 4 --reps 1 > gpurun_out/ncu_sweep.log 2>&1
fi
