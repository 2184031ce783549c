# timings for several shapes + ncu capture of the vote kernel (1 launch).
for a in "8 1000 200000" "3 1000 200000" "12 100 200000" "3 10 1000000"; do set -- $a
  python scripts/prof_vote.py --K $1 --C $2 --N $3 2>&1 | head -2; done > gpurun_out/prof_vote.txt
cat gpurun_out/prof_vote.txt
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vote_kernel -c 1 -o gpurun_out/$NCU \
  python scripts/prof_vote.py $NCU_ARGS --reps 1 > gpurun_out/ncu_vote.log 2>&1; echo ncu rc=$?
fi
