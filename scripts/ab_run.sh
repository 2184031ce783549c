#!/bin/bash
# Interleaved A/B of prebuilt librk variants (alt/*.so): scripts/ab_run.sh "K C N D REPS" ROUNDS name1 name2 ...
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
ARGS=$1; ROUNDS=$2; shift 2
for r in $(seq 1 $ROUNDS); do
  for v in "$@"; do
    echo "== $v round $r"
    RK_LIB=alt/$v.so timeout 300 python scripts/vote_reps.py $ARGS 2>&1 | tail -n +2 | awk "{print \$3}" | tr "\n" " "; echo
  done
done
