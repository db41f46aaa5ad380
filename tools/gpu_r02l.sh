set -x
mkdir -p gpurun_out
timeout 900 python tools/kernel_sweep.py --only srt19f32,srt19f32aa,trt19f32aa,cum19f32,cum19f32aa,srt19f64,srt19f64aa,cum19f64,cum19f64aa,srt27f32,srt27f32aa,cum27f32,cum27f32aa,srt27f64,srt27f64aa,cum27f64,cum27f64aa > gpurun_out/sweep_all.log 2>&1
for v in V0 V1; do
C="python tools/c3_node_level.py --ops srt19 --scen A --vars $v --steps 4 --warmup 2 --reps 1"
timeout 600 $C > gpurun_out/c3_srt19_$v.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 4 -c 1 -o gpurun_out/prof_srt19_$v $C > gpurun_out/ncu_srt19_$v.log 2>&1
done
