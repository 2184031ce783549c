#!/bin/bash
# --set full capture of the K = 8 averaging kernel (c4 shape) with source correlation
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
TAG=${1:-va}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vote_average -c 1 -o gpurun_out/${TAG} -f \
  python scripts/prof_vote.py --K 8 --C 1000 --N 200000 --gemm 2048 --reps 1 > gpurun_out/${TAG}.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_src.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
python scripts/vote_reps.py 8 1000 1000000 2048 5 > gpurun_out/${TAG}_reps.log 2>&1
tail -5 gpurun_out/${TAG}_reps.log
