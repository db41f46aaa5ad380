# collide sweep per variant library (alternated twice) with PSM_TMA=0, and the fp32 cumulant AA
# with PSM_TMA=1/2 on the current library
mkdir -p gpurun_out
ONLY=${ONLY:-srt19f32aa,cum19f32aa,cum27f32aa,cum27f32,srt27f32aa,srt19f64,cum19f64aa,cum27f64aa}
for r in 1 2; do
  for v in paper_2502_20049_b200/variants/*.so; do
    echo "== $(basename $v .so)" >> gpurun_out/tmaab.log
    PSM_TMA=0 PSM_LIB=$v timeout 600 python tools/kernel_sweep.py --only $ONLY >> gpurun_out/tmaab.log 2>&1
  done
  for t in 1 2; do
    echo "== b_new_tma$t" >> gpurun_out/tmaab.log
    PSM_TMA=$t PSM_LIB=paper_2502_20049_b200/variants/b_new.so timeout 600 python tools/kernel_sweep.py --only cum19f32aa,cum27f32aa >> gpurun_out/tmaab.log 2>&1
  done
done
