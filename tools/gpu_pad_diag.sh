# address sensitivity of the fp32 cumulant AA kernels: direction-plane padding sweep, old vs new
mkdir -p gpurun_out
for v in a_old b_new; do
  echo "== $v" >> gpurun_out/pad.log
  PSM_TMA=0 PSM_LIB=paper_2502_20049_b200/variants/$v.so timeout 900 python tools/kernel_sweep.py --only cum27f32aa,cum19f32aa --pads 0,32,64,256,1024,4096,65536 >> gpurun_out/pad.log 2>&1
done
