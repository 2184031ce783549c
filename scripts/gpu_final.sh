#!/bin/bash
# final verification: build, smoke, the whole -m gpu suite, bench lines of every config
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/final_smoke.log | tail -3
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final_tests.log
for c in c4 c5 c3 c2 c1; do
  timeout 900 python bench.py --config $c > gpurun_out/final_bench_$c.json 2> gpurun_out/final_bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --config c4 --fused --no-cpu-baseline > gpurun_out/final_bench_c4_fused.json 2> gpurun_out/final_bench_c4_fused.err; echo "fused rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc=$?"
