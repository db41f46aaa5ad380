mkdir -p gpurun_out
for round in 1 2; do
for v in paper_2502_20049_b200/variants/*.so; do
 for ab in 148 296; do
  echo "== $v ahead=$ab" >> gpurun_out/remapvar.log
  PSM_AHEAD_BLOCKS=$ab PSM_LIB=$v timeout 600 python tools/c3_node_level.py --ops srt27 --scen A --vars V3,V4 --steps 20 --reps 3 2>&1 | grep "^{" >> gpurun_out/remapvar.log
  PSM_AHEAD_BLOCKS=$ab PSM_LIB=$v timeout 300 python bench.py --config c5w --extra none --steps 20 --warmup 3 --reps 3 --no-cpu-baseline --no-e2e >> gpurun_out/remapvar.log 2>/dev/null
 done
done
done
