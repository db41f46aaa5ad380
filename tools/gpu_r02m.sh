set -x
mkdir -p gpurun_out
timeout 900 python tools/kernel_sweep.py --only srt19f32,srt19f32aa,trt19f32aa,cum19f32,cum19f32aa,srt19f64,srt19f64aa,cum19f64,cum19f64aa,srt27f32,srt27f32aa,cum27f32,cum27f32aa,srt27f64,srt27f64aa,cum27f64,cum27f64aa > gpurun_out/sweep_all.log 2>&1
rm -f gpurun_out/bench_next.jsonl
for c in c5w c5wpap c5wcum c5w64 c4aa; do
  timeout 300 python bench.py --config $c --extra none --steps 20 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/$c /" >> gpurun_out/bench_next.jsonl 2>> gpurun_out/bench_next.err
done
