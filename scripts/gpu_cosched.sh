#!/bin/bash
# co-scheduling probe: GEMM (half of c4) concurrent with the vote stage of the other half, per GEMM
# stage-count variant (alt/*.so from scripts/ab_build.sh) and averaging CTAs per SM
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
VARIANTS="${VARIANTS:-ns6 ns5c ns4c ns3c}" PER_SM="${PER_SM:-6 2 1}" bash scripts/cosched_sweep.sh 2>&1 | tee gpurun_out/cosched.log
