mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l3_V4b.csv python tools/c3_node_level.py --ops cum19aa --scen A --vars V4 --steps 4 --warmup 1 --reps 1 > /dev/null 2>&1
V=V4 K=k_remap_l3_mesh bash tools/gpu_remap_ncu.sh
