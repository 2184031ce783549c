#!/bin/bash
# A/B of prebuilt librk variants (alt/*.so, same exports): vote-only reps and bench; parity tests on the in-tree build
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -m gpu -x ${TESTS:-tests/test_gpu_multiwave.py tests/test_gpu_vote.py tests/test_gpu_offsets.py} > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_tests.log
for r in 1 2 3; do for v in $VARIANTS; do
  echo "== $v round $r (vote only)"; RK_LIB=alt/$v.so timeout 300 python scripts/vote_reps.py ${SHAPE:-8 1000 1000000 2048} 4 v 2>&1 | tail -4 | awk '{print $3}' | tr "\n" " "; echo
done; done
for v in $VARIANTS; do
  echo "== $v bench"; RK_LIB=alt/$v.so timeout 600 python bench.py --no-cpu-baseline --steps 10 ${BENCH_ARGS} > gpurun_out/ab_bench_$v.json 2>gpurun_out/ab_bench_$v.err; python -c "
import json; d=json.load(open('gpurun_out/ab_bench_$v.json')); print(d['ms_per_step'], {k: round(v, 3) for k, v in d['kernels_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
done
