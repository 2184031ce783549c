#!/bin/bash
# NEXT-3 check: build, fused tests, fused vs unfused bench lines (c4, c3)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_fused.py > gpurun_out/fused_tests.log 2>&1
rc=$?
tail -30 gpurun_out/fused_tests.log
for c in c4 c3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_fused.json 2> gpurun_out/bench_${c}_fused.err; tail -c 1500 gpurun_out/bench_${c}_fused.json; tail -3 gpurun_out/bench_${c}_fused.err
  timeout 600 python bench.py --config $c --no-cpu-baseline --unfused > gpurun_out/bench_${c}_unfused.json 2> gpurun_out/bench_${c}_unfused.err; tail -c 600 gpurun_out/bench_${c}_unfused.json
done
exit $rc
