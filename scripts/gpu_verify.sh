#!/bin/bash
# final verification: build, full -m gpu suite, smoke, compute-sanitizer (all tools), bench c4 / c5
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gpu_tests.log 2>&1
rc=$?
tail -14 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for tool in memcheck racecheck synccheck; do
  for w in c1 c2 k12 fused serve rl; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py $w > gpurun_out/san_${tool}_${w}.log 2>&1
    echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_${w}.log | tail -1)"
  done
done
for c in c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
exit $rc
