#!/bin/bash
# row-skip A/B (RK_NO_ROW_SKIP) in one build + the GEMM/vote parity tests
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_multiwave.py tests/test_gpu_gemm.py tests/test_gpu_vote.py tests/test_gpu_offsets.py tests/test_gpu_fullsize.py tests/test_gpu_fused.py > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab_tests.log
for r in 1 2 3; do for v in noskip skip; do
  if [ $v = noskip ]; then export RK_NO_ROW_SKIP=1; else unset RK_NO_ROW_SKIP; fi
  echo "== $v round $r (vote only)"; timeout 300 python scripts/vote_reps.py 8 1000 1000000 2048 4 v 2>&1 | tail -4 | awk '{print $3, $6}' | tr "\n" " "; echo
done; done
for v in noskip skip; do
  if [ $v = noskip ]; then export RK_NO_ROW_SKIP=1; else unset RK_NO_ROW_SKIP; fi
  echo "== $v bench"; timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ab_bench_$v.json 2>gpurun_out/ab_bench_$v.err; python -c "
import json; d=json.load(open('gpurun_out/ab_bench_$v.json')); print(d['ms_per_step'], d['kernels_ms_per_step'], d['vote_stage'].get('frac_dram'), d['vote_stage'].get('rows_skipped_frac'), d['clocks'])"
done
