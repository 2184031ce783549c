# ncu --set full of the K=12 (c5-shape) vote kernels, GEMM-fed, N = 1M.
timeout 900 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-vote_} -c ${NCU_COUNT:-3} -o gpurun_out/k12 \
  python scripts/prof_vote.py --K 12 --C 100 --N 1000000 --gemm 1024 --reps 1 > gpurun_out/k12.log 2>&1
echo "k12 rc=$?"
