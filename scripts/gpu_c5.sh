#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
R=r02
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vote -c 5 -o gpurun_out/${R}_k12 -f \
  python scripts/prof_vote.py --K 12 --C 100 --N 250000 --gemm 1024 --reps 1 > gpurun_out/${R}_k12.log 2>&1
echo "k12 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_heads -c 1 -o gpurun_out/${R}_gemm12 -f \
  python scripts/prof_vote.py --K 12 --C 100 --N 131072 --gemm 1024 --reps 1 > gpurun_out/${R}_gemm12.log 2>&1
echo "gemm12 rc=$?"
timeout 900 python bench.py --config c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
