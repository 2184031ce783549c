# GPU check used during development: smoke + GPU parity tests (logs under gpurun_out/).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 ${PYTEST_ARGS} 2>&1 | tail -80 > gpurun_out/gpu_tests.log; echo tests done
tail -3 gpurun_out/smoke.log
cat gpurun_out/gpu_tests.log
