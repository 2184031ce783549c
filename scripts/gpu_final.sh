#!/bin/bash
# round-end check: build, full -m gpu suite, smoke, racecheck of the GEMM drivers, bench lines
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1
rc=$?
tail -25 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
for w in c1 c2 fused serve; do
  timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_run.py $w > gpurun_out/san_racecheck_${w}.log 2>&1
  echo "racecheck $w rc=$? $(grep -E 'RACECHECK SUMMARY' gpurun_out/san_racecheck_${w}.log | tail -1)"
done
for c in c4 c5 c3 c2; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --config c4 --fused --no-cpu-baseline > gpurun_out/bench_c4_fused.json 2> gpurun_out/bench_c4_fused.err; echo "bench c4 fused rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
exit $rc
