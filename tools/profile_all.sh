#!/usr/bin/env bash
# One GPU call: the bench line, the bench-step launch list and the ncu --set full
# captures behind profiles/ (summarised here afterwards by tools/profile_summary.py).
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
tail -1 gpurun_out/bench_full.log > gpurun_out/bench_line.json
export QLRT_NO_TORCH_PROFILER=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1
N="--set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 ncu $N -k regex:"gemm_kernel<.int.512, .bool.1" -s 2 -c 2 -o gpurun_out/prof_fused_c2 \
  python tools/prof_driver.py gemm_bwd > /dev/null 2>&1
timeout 600 ncu $N -k regex:"gemm_kernel<.int.512, .bool.1" -s 2 -c 1 -o gpurun_out/prof_fused_gu \
  python tools/prof_driver.py gemm_gu > /dev/null 2>&1
timeout 300 ncu $N -k regex:dequant64_bf16 -s 2 -c 1 -o gpurun_out/prof_dequant_c1 python tools/prof_driver.py dequant > /dev/null 2>&1
timeout 300 ncu $N -k regex:"quantize64|dq_chunk|dq_encode" -s 3 -c 3 -o gpurun_out/prof_quantize_c1 python tools/prof_driver.py quantize > /dev/null 2>&1
timeout 300 ncu $N -k regex:gemv_mma -s 2 -c 1 -o gpurun_out/prof_gemv_c4 python tools/prof_driver.py gemv > /dev/null 2>&1
ls -la gpurun_out/
