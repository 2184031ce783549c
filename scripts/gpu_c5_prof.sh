#!/bin/bash
# c5 per-kernel launch list (ncu durations) + full captures of the packed GEMM and the K = 12 classify kernel
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv \
  python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c5_ncu_bench.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_heads -c 1 -o gpurun_out/c5_gemm -f \
  python scripts/prof_vote.py --K 12 --C 100 --N 131072 --gemm 1024 --reps 1 > gpurun_out/c5_gemm.log 2>&1
echo "gemm rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vote_group_classify -c 1 -o gpurun_out/c5_gc -f \
  python scripts/prof_vote.py --K 12 --C 100 --N 250000 --gemm 1024 --reps 1 > gpurun_out/c5_gc.log 2>&1
echo "gc rc=$?"
