set -x
mkdir -p gpurun_out
C="python tools/c3_node_level.py --ops srt27 --scen A --vars V4 --steps 4 --warmup 2 --reps 1"
timeout 600 $C > gpurun_out/c3A4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_remap_l3_chunks -s 6 -c 1 -o gpurun_out/prof_l3chunks $C > gpurun_out/ncu_l3c.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_remap_l2 -s 6 -c 1 -o gpurun_out/prof_l2 $C > gpurun_out/ncu_l2.log 2>&1
PSM_MAP_STATS=1 timeout 600 $C > gpurun_out/c3A4_stats.log 2>&1
