# which AA kernel of the fp32 D3Q27 cumulant depends on the library build: launch lists and a
# full ncu of the even and odd launches, old vs new library
mkdir -p gpurun_out
for v in a_old b_new; do
  PSM_TMA=0 PSM_LIB=paper_2502_20049_b200/variants/$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/odd_launch_$v.csv python tools/kernel_sweep.py --only cum27f32aa --steps 6 --reps 1 > /dev/null 2>&1
  PSM_TMA=0 PSM_LIB=paper_2502_20049_b200/variants/$v.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_collide -s 6 -c 2 -o gpurun_out/odd_prof_$v python tools/kernel_sweep.py --only cum27f32aa --steps 6 --reps 1 > /dev/null 2>&1
done
