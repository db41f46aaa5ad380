# remap knobs on c3 scenario A (cum19aa, V3 = s1, V4 = s2): cached band at s = 2, persistent
# block counts of the remap-ahead kernels; plus the new band-pass face test
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "faces or cror_rotor" > gpurun_out/knobs_tests.log 2>&1; echo "rc=$?" >> gpurun_out/knobs_tests.log
C3="tools/c3_node_level.py --ops cum19aa --scen A --steps 20 --reps 3"
for r in 1 2; do
  echo "== default" >> gpurun_out/knobs.log; timeout 300 python $C3 --vars V3,V4 2>&1 | grep "^{" >> gpurun_out/knobs.log
  echo "== cache_s2" >> gpurun_out/knobs.log; PSM_CACHE_MAX_S=2 timeout 300 python $C3 --vars V4 2>&1 | grep "^{" >> gpurun_out/knobs.log
  for nb in 148 296 444 592; do
    echo "== blocks$nb" >> gpurun_out/knobs.log; PSM_AHEAD_BLOCKS=$nb timeout 300 python $C3 --vars V3,V4 2>&1 | grep "^{" >> gpurun_out/knobs.log
  done
done
