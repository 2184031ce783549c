# ncu captures of the vote kernel for several shapes (1 launch each)
i=0
for a in "$@"; do i=$((i+1))
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:vote -c ${NCU_COUNT:-1} -o gpurun_out/vote_p$i \
    python scripts/prof_vote.py $a --reps 1 > gpurun_out/ncu_p$i.log 2>&1; echo "p$i [$a] rc=$?"
done
