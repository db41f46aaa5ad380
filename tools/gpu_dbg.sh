set -x
timeout 300 python bench.py --config c5wr2 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_r2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2.csv python bench.py --config c5wr2 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r2.log 2>&1
