#!/bin/bash
# bench-only A/B of prebuilt librk variants: CONFIGS x ROUNDS x VARIANTS, interleaved
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest -q -m gpu -x $TESTS > gpurun_out/abb_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/abb_tests.log; fi
for c in ${CONFIGS:-c4}; do for r in $(seq 1 ${ROUNDS:-2}); do for v in $VARIANTS; do
  RK_LIB=alt/$v.so timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/abb_${c}_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/abb_${c}_$v.json')); ks=d['kernels_ms_per_step']; print('$c $v', round(d['ms_per_step'], 3), 'kernels', round(sum(ks.values()), 3), {k: round(v, 3) for k, v in ks.items()}, d['clocks']['sm_mhz'])"
done; done; done
