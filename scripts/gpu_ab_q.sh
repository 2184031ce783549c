#!/bin/bash
# labelled-moments A/B (packed two-rate multiply-adds vs RK_Q_UNPACKED) + nested-vs-generic check + c5 parity
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python scripts/q_check.py 2>&1 | tail -6
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_multiwave.py tests/test_gpu_vote.py > gpurun_out/abq_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/abq_tests.log
for r in 1 2; do for v in unpacked packed; do
  if [ $v = unpacked ]; then export RK_Q_UNPACKED=1; else unset RK_Q_UNPACKED; fi
  timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 10 > gpurun_out/abq_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/abq_$v.json')); print('$v', round(d['ms_per_step'], 3), {k: round(v, 3) for k, v in d['kernels_ms_per_step'].items()})"
done; done
