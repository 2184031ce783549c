# Round profiling: (1) launch list of the bench command (c4), (2) --set full of the GEMM,
# (3) of the K=8 vote kernels, (4) of the K=12 vote kernels (c5 shape).
R=${ROUND:-r02}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
  python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${R}_launches_bench.json 2> gpurun_out/${R}_launches.err
echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_heads -c 1 -o gpurun_out/${R}_gemm \
  python scripts/prof_vote.py --K 8 --C 1000 --N 65536 --gemm 2048 --reps 1 > gpurun_out/${R}_gemm.log 2>&1
echo "gemm rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vote -c 2 -o gpurun_out/${R}_vote \
  python scripts/prof_vote.py --K 8 --C 1000 --N 200000 --gemm 2048 --reps 1 > gpurun_out/${R}_vote.log 2>&1
echo "vote rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vote -c 5 -o gpurun_out/${R}_k12 \
  python scripts/prof_vote.py --K 12 --C 100 --N 250000 --gemm 1024 --reps 1 > gpurun_out/${R}_k12.log 2>&1
echo "k12 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_heads -c 1 -o gpurun_out/${R}_gemm12 \
  python scripts/prof_vote.py --K 12 --C 100 --N 131072 --gemm 1024 --reps 1 > gpurun_out/${R}_gemm12.log 2>&1
echo "gemm12 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_heads|vote_sparse|vote_classify|gather_rows|vote_average" -c 6 -o gpurun_out/${R}_fused \
  python scripts/prof_fused.py --N 131072 --reps 1 > gpurun_out/${R}_fused.log 2>&1
echo "fused rc=$?"
