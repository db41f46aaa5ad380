# fused L1+L2 remap launch: remap GPU tests (fused default, then the two-launch path), then
# c3 scenario A (R1, s = 1/2) and c5w with PSM_REMAP_L12=0/1 alternated; then the c5wpap
# occupancy check (tools/gpu_hiocc_pap.sh)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "mesh or seam or voxel or rotor or propeller or fullsize or faces or table1 or R2" > gpurun_out/l12_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/l12_tests.log
PSM_REMAP_L12=0 timeout 900 python -m pytest tests/test_gpu_seam.py -x -q > gpurun_out/l12_tests0.log 2>&1; echo "tests rc=$?" >> gpurun_out/l12_tests0.log
for r in 1 2; do for f in 0 1; do
  echo "== l12_$f" >> gpurun_out/l12.log
  PSM_REMAP_L12=$f timeout 600 python tools/c3_node_level.py --ops cum19aa --scen A --vars V3,V4 --steps 20 --reps 3 2>&1 | grep "^{" >> gpurun_out/l12.log
  PSM_REMAP_L12=$f timeout 400 python bench.py --config c5w --extra none --steps 20 --warmup 3 --reps 3 --no-cpu-baseline --no-e2e >> gpurun_out/l12.log 2>&1
done; done
bash tools/gpu_hiocc_pap.sh
