mkdir -p gpurun_out
for v in V3 V4; do
PSM_MAP_STATS=1 timeout 300 python tools/c3_node_level.py --ops cum19aa --scen A --vars $v --steps 2 --warmup 1 --reps 1 > gpurun_out/stats_$v.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l3_$v.csv python tools/c3_node_level.py --ops cum19aa --scen A --vars $v --steps 4 --warmup 1 --reps 1 > gpurun_out/l3ncu_$v.log 2>&1
done
