mkdir -p gpurun_out
for r in 1 2; do
echo "== default" >> gpurun_out/r2c.log
timeout 300 python tools/c3_node_level.py --ops cum19aa --scen A --vars V3,V4 --steps 20 --reps 3 --mapping R2 2>&1 | grep "^{" >> gpurun_out/r2c.log
echo "== cache3" >> gpurun_out/r2c.log
PSM_CACHE_MAX_S=3 timeout 300 python tools/c3_node_level.py --ops cum19aa --scen A --vars V3,V4 --steps 20 --reps 3 --mapping R2 2>&1 | grep "^{" >> gpurun_out/r2c.log
done
