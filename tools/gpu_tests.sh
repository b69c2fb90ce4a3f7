#!/usr/bin/env bash
# one gpurun call: smoke + GPU parity tests with hard timeouts
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q --timeout 240 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/smoke.log; tail -40 gpurun_out/pytest_gpu.log
