mkdir -p gpurun_out
V=${V:-V4}; K=${K:-k_remap_l3_chunks}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s 8 -c 1 -o gpurun_out/remap_$V python tools/c3_node_level.py --ops cum19aa --scen A --vars $V --steps 4 --warmup 1 --reps 1 > gpurun_out/remap_ncu_$V.log 2>&1
ncu -i gpurun_out/remap_$V.ncu-rep --page raw --csv > gpurun_out/remap_${V}_raw.csv 2>&1
ncu -i gpurun_out/remap_$V.ncu-rep --page source --csv > gpurun_out/remap_${V}_src.csv 2>&1
