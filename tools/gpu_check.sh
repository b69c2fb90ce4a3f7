#!/usr/bin/env bash
# one gpurun call: GPU tests (optionally a subset) + a bench run; logs under gpurun_out/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q --timeout 300 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
if [ -n "${BENCH:-1}" ] && [ "${BENCH:-1}" != "0" ]; then
  timeout ${BENCH_TIMEOUT:-900} python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench exit $?" >> gpurun_out/bench.err
  tail -5 gpurun_out/bench.err
  cat gpurun_out/bench.json
fi
