set -x
for cfg in "148 256" "296 128" "592 64" "148 128" "148 64" "74 256"; do set -- $cfg; PSM_AHEAD_BLOCKS=$1 PSM_AHEAD_THREADS=$2 timeout 300 python bench.py --config c5w --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ab_$1_$2.json 2> gpurun_out/bench_ab_$1_$2.err; done
