# A/B of the libraries under paper_2502_20049_b200/variants/ (alternated twice): the remap-
# related GPU tests on the current library first, then c5w bench and c3 scenario A per library
mkdir -p gpurun_out
export PSM_VOXELIZE_CHECK=1
timeout 900 python -m pytest tests -x -q -m gpu -k "${TESTK:-mesh or seam or voxel or rotor or propeller or fullsize or faces}" > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
unset PSM_VOXELIZE_CHECK
for r in 1 2; do for v in paper_2502_20049_b200/variants/*.so; do
  echo "== $(basename $v .so)" >> gpurun_out/ab.log
  PSM_LIB=$v timeout 400 python bench.py --extra c5w --no-cpu-baseline --no-e2e --reps 3 >> gpurun_out/ab.log 2>&1
  PSM_LIB=$v timeout 600 python tools/c3_node_level.py --ops ${C3OPS:-srt27,cum19aa} --scen A --vars ${C3VARS:-V3,V4} --steps 20 --reps 3 2>&1 | grep "^{" >> gpurun_out/ab.log
done; done
