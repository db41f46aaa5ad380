# R2 (paper-literal centre-only mapping) block count by popcount masks: parity tests, then the
# c3 node-level variants with R1 and R2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "faces or R2 or seam or table1" > gpurun_out/r2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_tests.log
for m in R1 R2; do
  echo "== $m" >> gpurun_out/r2.log
  timeout 900 python tools/c3_node_level.py --ops cum19aa --scen A,B --vars V0,V1,V2,V3,V4 --steps 20 --reps 3 --mapping $m 2>&1 | grep "^{" >> gpurun_out/r2.log
done
