# ncu evidence for profiles/ (one GPU; each capture only after the same command ran cleanly):
#   gpurun --timeout 2400 -- 'bash tools/gpu_profile.sh'
# then: python tools/ncu_summary.py gpurun_out/prof_c5w.ncu-rep c5w 134217728 152
#       python tools/ncu_details.py gpurun_out/prof_c5w.ncu-rep "<header>" > profiles/rNN_ncu_c5w_collide.txt
#       python tools/launch_table.py gpurun_out/launches_c5w.csv "<cmd>" 5 > profiles/rNN_launches_c5w.txt
set -x
mkdir -p gpurun_out
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/plain_c5w.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 5 -c 1 -o gpurun_out/prof_c5w $B > gpurun_out/ncu_c5w.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_remap_l3 -s 3 -c 1 -o gpurun_out/prof_c5w_remap $B > gpurun_out/ncu_c5w_remap.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_c5w5.log 2>&1 && \
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5w.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
