# Additional ncu captures for profiles/ (one GPU): AA odd/even collide, cumulant fp64, the
# incremental remap over the cached band.
set -x
mkdir -p gpurun_out
A="python bench.py --config c4aa --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $A > gpurun_out/plain_aa.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 5 -c 2 -o gpurun_out/prof_c4aa $A > gpurun_out/ncu_aa.log 2>&1
C="python bench.py --config c3cum --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $C > gpurun_out/plain_cum3.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 5 -c 1 -o gpurun_out/prof_c3cum $C > gpurun_out/ncu_cum3.log 2>&1
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/plain_c5w.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_remap_l3 -s 8 -c 1 -o gpurun_out/prof_c5w_band $B > gpurun_out/ncu_band.log 2>&1
