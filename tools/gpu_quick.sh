set -x
rm -f gpurun_out/bench_abl.jsonl
for rep in 1 2; do for v in b3 b4; do cp abtest/libpsm_$v.so paper_2502_20049_b200/libpsm.so; timeout 300 python bench.py --config c4aa --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/c4aa-$v /" >> gpurun_out/bench_abl.jsonl 2>> gpurun_out/bench_abl.err; done; done
cp abtest/libpsm_b3.so paper_2502_20049_b200/libpsm.so
