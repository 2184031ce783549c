#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_fused.py > gpurun_out/fused_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/fused_tests.log
python scripts/prof_fused.py --N 1000000 --reps 3
python scripts/prof_fused.py --N 1000000 --reps 3 --unfused
