set -x
mkdir -p gpurun_out
timeout 600 python tools/kernel_sweep.py > gpurun_out/sweep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:k_collide --csv --log-file gpurun_out/sweep_ncu.csv python tools/kernel_sweep.py --steps 4 --reps 1 > gpurun_out/sweep_ncu.log 2>&1
