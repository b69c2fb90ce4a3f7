#!/usr/bin/env bash
# tests + smoke + bench in one gpurun call
cd "$(dirname "$0")/.."
bash tools/gpu_tests.sh > /dev/null 2>&1
timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
tail -5 gpurun_out/smoke.log; tail -25 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
