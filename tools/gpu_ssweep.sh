# super-sampling sweep of the c5w rotor pair (fp32), with and without the remap-ahead overlap:
#   gpurun --timeout 1800 -- 'bash tools/gpu_ssweep.sh'
set -x
mkdir -p gpurun_out
rm -f gpurun_out/ssweep.jsonl
for s in 0 1 2 3; do timeout 300 python bench.py --config c5w --extra none --s $s --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/s$s /" >> gpurun_out/ssweep.jsonl 2>> gpurun_out/ssweep.err; done
for s in 0 1 2 3; do PSM_NO_REMAP_AHEAD=1 timeout 300 python bench.py --config c5w --extra none --s $s --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/s$s-serial /" >> gpurun_out/ssweep.jsonl 2>> gpurun_out/ssweep.err; done
# the paper's literal centre-only mapping (R2, reading A12) on the same rotor pair
for s in 0 1 2 3; do timeout 300 python bench.py --config c5wr2 --extra none --s $s --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/s$s-r2 /" >> gpurun_out/ssweep.jsonl 2>> gpurun_out/ssweep.err; done
