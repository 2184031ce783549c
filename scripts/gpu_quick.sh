#!/bin/bash
# quick GPU check of selected test files: build + pytest on the given args
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest -q -m gpu "$@" > gpurun_out/quick_tests.log 2>&1
rc=$?
tail -30 gpurun_out/quick_tests.log
exit $rc
