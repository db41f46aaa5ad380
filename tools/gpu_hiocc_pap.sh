# occupancy choice for the paper configuration (c5wpap) and the default line: PSM_HIOCC=0/1
mkdir -p gpurun_out
for r in 1 2; do for h in 0 1; do
  echo "== hiocc$h" >> gpurun_out/hiocc_pap.log
  for c in c5wpap c5w64; do
    PSM_HIOCC=$h timeout 300 python bench.py --config $c --extra none --steps 20 --warmup 3 --reps 3 --no-cpu-baseline --no-e2e >> gpurun_out/hiocc_pap.log 2>&1
  done
done; done
PSM_MAP_STATS=1 timeout 300 python bench.py --config c5wpap --extra none --steps 3 --warmup 3 --reps 1 --no-cpu-baseline --no-e2e 2>&1 | grep "psm step" | tail -2 >> gpurun_out/hiocc_pap.log
