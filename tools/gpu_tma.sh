# TMA-staged AA even step (fp32 cumulant): parity tests with PSM_TMA=1 and 2, then the AA
# cumulant sweep per library / TMA mode, alternated
mkdir -p gpurun_out
for t in 1 2; do
PSM_TMA=$t timeout 900 python -m pytest tests -x -q -m gpu -k "aa or AA or cumulant or paper or pattern" > gpurun_out/tma_tests$t.log 2>&1; echo "tests rc=$?" >> gpurun_out/tma_tests$t.log
done
ONLY=cum19f32aa,cum27f32aa,srt19f32aa
for r in 1 2; do
  echo "== old" >> gpurun_out/tma.log
  PSM_LIB=paper_2502_20049_b200/variants/a_old.so timeout 600 python tools/kernel_sweep.py --only $ONLY >> gpurun_out/tma.log 2>&1
  for t in 0 1 2; do
    echo "== tma$t" >> gpurun_out/tma.log
    PSM_TMA=$t timeout 600 python tools/kernel_sweep.py --only $ONLY >> gpurun_out/tma.log 2>&1
  done
done
PSM_TMA=2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_tma2.csv python tools/kernel_sweep.py --only cum27f32aa --steps 6 --reps 1 > /dev/null 2>&1
