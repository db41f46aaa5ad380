set -x
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/plain_c5w.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 5 -c 1 -o gpurun_out/prof_c5w_final $B > gpurun_out/ncu_c5w.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_remap_l3 -s 3 -c 1 -o gpurun_out/prof_c5w_remap $B > gpurun_out/ncu_c5w_remap.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5w.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
C="python bench.py --config c5wcum --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $C > gpurun_out/plain_cum.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 5 -c 1 -o gpurun_out/prof_c5wcum_final $C > gpurun_out/ncu_cum.log 2>&1
D="python bench.py --config c5app --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $D > gpurun_out/plain_app.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 5 -c 1 -o gpurun_out/prof_c5app_final $D > gpurun_out/ncu_app.log 2>&1
