#!/bin/bash
# exceed-time prefix sums vs the per-batch sweep (RK_E_SWEEP): parity tests + c5 / c4 bench A/B
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest -q -m gpu -x tests/test_gpu_vote.py tests/test_gpu_multiwave.py tests/test_gpu_arrivals.py tests/test_gpu_offsets.py tests/test_gpu_fullsize.py tests/test_gpu_multiproc.py > gpurun_out/abe_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/abe_tests.log
for c in c5 c4; do for r in 1 2; do for v in sweep psum; do
  if [ $v = sweep ]; then export RK_E_SWEEP=1; else unset RK_E_SWEEP; fi
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/abe_${c}_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/abe_${c}_$v.json')); print('$c $v', round(d['ms_per_step'], 3), {k: round(v, 3) for k, v in d['kernels_ms_per_step'].items()})"
done; done; done
