#!/bin/bash
# host-X (e2e) path: GPU tests that stage host inputs, then bench lines of c4 / c5 / c4 fused
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/e2e_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/e2e_tests.log
for c in c4 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/e2e_bench_$c.json 2> gpurun_out/e2e_bench_$c.err; echo "bench $c rc=$?"; tail -2 gpurun_out/e2e_bench_$c.err
done
timeout 900 python bench.py --config c4 --fused --no-cpu-baseline > gpurun_out/e2e_bench_c4f.json 2> gpurun_out/e2e_bench_c4f.err; echo "bench c4f rc=$?"; tail -2 gpurun_out/e2e_bench_c4f.err
