# ncu --set full of the labelled-moments kernel at the c5 shape (K=12, 4095 subsets).
timeout 600 ncu --set full --import-source on --clock-control none -k regex:q_kernel -c 1 -o gpurun_out/q_c5 \
  python scripts/prof_vote.py --K 12 --C 100 --N 4000000 --gemm 1024 --reps 1 > gpurun_out/q_c5.log 2>&1
echo "q rc=$?"
