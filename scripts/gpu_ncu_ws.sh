#!/bin/bash
# full capture (with source) of the K = 12 warp-per-sample averaging kernel, first pass
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vote_wsample_average -c 1 -o gpurun_out/c5_ws -f \
  python scripts/prof_vote.py --K 12 --C 100 --N 250000 --gemm 1024 --reps 1 > gpurun_out/c5_ws.log 2>&1
echo "ws rc=$?"
