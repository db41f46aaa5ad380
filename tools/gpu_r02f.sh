# round-2 measurement batch (1 GPU): collide sweep of every operator/stencil/precision/pattern,
# the c3 node-level table, AA ncu evidence, and the NEXT-row bench workloads
set -x
mkdir -p gpurun_out
timeout 900 python tools/kernel_sweep.py --only srt19f32,srt19f32aa,trt19f32,trt19f32aa,cum19f32,cum19f32aa,srt19f64,srt19f64aa,trt19f64,cum19f64,cum19f64aa,srt27f32,srt27f32aa,cum27f32,cum27f32aa,srt27f64,srt27f64aa,cum27f64,cum27f64aa > gpurun_out/sweep_all.log 2>&1
timeout 1500 python tools/c3_node_level.py --out gpurun_out/r02_c3_node_level.md --json gpurun_out/r02_c3_node_level.json > gpurun_out/c3.log 2>&1
S="python tools/kernel_sweep.py --only cum19f64aa,srt19f32aa,cum27f32aa --steps 4 --reps 1"
timeout 300 $S > gpurun_out/plain_sweep.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 6 -c 2 -o gpurun_out/prof_aa_cum19f64 $S > gpurun_out/ncu_aa1.log 2>&1
rm -f gpurun_out/bench_next.jsonl
for c in c5wpap c5wcum c5w27 c4aa c4f64 c4trt c3cum c3f64 c5wr2 c4; do
  timeout 300 python bench.py --config $c --extra none --steps 20 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/$c /" >> gpurun_out/bench_next.jsonl 2>> gpurun_out/bench_next.err
done
