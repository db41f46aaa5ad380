# Full single-GPU check (run through gpurun from the repo root):
#   gpurun --timeout 3000 -- 'bash tools/gpu_check.sh'
# GPU tests, the default bench line, every bench workload, and the no-remap-ahead variant.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
rm -f gpurun_out/bench_all.jsonl
for c in c5app c5wr2 c5w27 c5wcum c4 c4aa c4f64 c4trt c4dyn c3f64 c3cum; do
  timeout 300 python bench.py --config $c --steps 40 --warmup 3 --no-cpu-baseline | sed "s/^/$c /" >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err
done
PSM_NO_REMAP_AHEAD=1 timeout 300 python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e | sed "s/^/c5w-noahead /" >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_n1.json 2> gpurun_out/ref_n1.err
