#!/bin/bash
# GEMM-only A/B of prebuilt librk variants (alt/*.so) at a shape, interleaved; GEMM parity tests on each
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for v in $VARIANTS; do
  RK_LIB=alt/$v.so timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_gemm.py tests/test_gpu_multiwave.py > gpurun_out/abg_tests_$v.log 2>&1; echo "$v tests rc=$?"; tail -1 gpurun_out/abg_tests_$v.log
done
for r in 1 2 3; do for v in $VARIANTS; do
  echo "== $v round $r: $(RK_LIB=alt/$v.so timeout 300 python scripts/prof_gemm.py ${GSHAPE:---K 12 --C 100 --D 1024 --N 2000000} --reps 5 2>&1 | tail -1)"
done; done
for v in $VARIANTS; do
  echo "== $v bench"; RK_LIB=alt/$v.so timeout 600 python bench.py --no-cpu-baseline --steps 10 ${BENCH_ARGS} > gpurun_out/ab_bench_$v.json 2>gpurun_out/ab_bench_$v.err; python -c "
import json; d=json.load(open('gpurun_out/ab_bench_$v.json')); print(d['ms_per_step'], {k: round(v, 3) for k, v in d['kernels_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
done
