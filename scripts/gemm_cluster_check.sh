# correctness + timing of the head GEMM at cluster 1 and 2 (short timeouts: a barrier bug would hang)
for cl in 2 1; do
  echo "== RK_GEMM_CLUSTER=$cl"
  RK_GEMM_CLUSTER=$cl timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
  RK_GEMM_CLUSTER=$cl timeout 300 python scripts/prof_vote.py --K 8 --C 1000 --N 1000000 --gemm 2048 --reps 3 2>&1 | grep -E "gemm|vote " | head -3
done
