# Development bench run (logs under gpurun_out/).
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
for c in ${CONFIGS:-c4}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
  cat gpurun_out/bench_$c.json; tail -5 gpurun_out/bench_$c.err
done
