#!/bin/bash
# ncu launch lists (durations only) of bench.py for the given configs: CONFIGS="c4 c4f" (c4f = c4 --fused)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in ${CONFIGS:-c4}; do
  args="--config ${c%f}"; [ "${c%f}" != "$c" ] && args="$args --fused"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$c.csv \
    python bench.py $args --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ll_$c.log 2>&1
  echo "$c rc=$?"
done
