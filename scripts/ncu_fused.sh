#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:"gemm_heads_kernel|vote_sparse" -c 2 -o gpurun_out/fused_full2 -f python scripts/prof_fused.py --N 131072 --reps 1 > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/ncu_fused.log
