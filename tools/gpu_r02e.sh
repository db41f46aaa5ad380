set -x
mkdir -p gpurun_out
C="python tools/c3_node_level.py --ops srt27 --scen A --vars V1,V3,V4 --steps 6 --warmup 3 --reps 1"
timeout 600 $C > gpurun_out/c3A_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3A_launches.csv $C > gpurun_out/c3A_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 40 -c 1 -o gpurun_out/prof_c3A_V1 python tools/c3_node_level.py --ops srt27 --scen A --vars V1 --steps 6 --warmup 3 --reps 1 > gpurun_out/c3A_full.log 2>&1
timeout 600 python tools/kernel_sweep.py --only srt27f32aa,cum27f32,cum27f32aa > gpurun_out/sweep.log 2>&1
timeout 600 python bench.py --config c5wcum --extra none --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5wcum.json 2> gpurun_out/bench_c5wcum.err
timeout 600 python bench.py --config c5wpap --extra none --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5wpap.json 2> gpurun_out/bench_c5wpap.err
