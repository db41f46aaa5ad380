# fp32 cumulant AA kernels (D3Q27 87.6 %, D3Q19 92.8 %): launch list (even/odd split) and an
# ncu --set full of one even and one odd launch of each
mkdir -p gpurun_out
for v in cum27f32aa cum19f32aa; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$v.csv python tools/kernel_sweep.py --only $v --steps 6 --reps 1 > /dev/null 2>&1
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_collide -s 6 -c 2 -o gpurun_out/prof_$v python tools/kernel_sweep.py --only $v --steps 6 --reps 1 > gpurun_out/ncu_$v.log 2>&1
done
