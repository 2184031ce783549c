#!/bin/bash
# round-2 GPU check: build, full -m gpu suite, smoke, bench lines
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q --durations=25 "$@" > gpurun_out/gpu_tests.log 2>&1
rc=$?
tail -40 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -1 gpurun_out/bench_c4.json
timeout 600 python bench.py --config c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -1 gpurun_out/bench_c5.json
exit $rc
