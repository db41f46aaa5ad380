set -x
for rep in 1 2; do for v in base CS LU; do cp abtest/libpsm_$v.so paper_2502_20049_b200/libpsm.so; PSM_NO_REMAP_AHEAD=1 timeout 300 python bench.py --config c5w --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/$v /" >> gpurun_out/bench_abl.jsonl 2>> gpurun_out/bench_abl.err; done; done
for v in base CS; do cp abtest/libpsm_$v.so paper_2502_20049_b200/libpsm.so; timeout 300 python bench.py --config c4 --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/c4$v /" >> gpurun_out/bench_abl.jsonl 2>> gpurun_out/bench_abl.err; done
cp abtest/libpsm_base.so paper_2502_20049_b200/libpsm.so
