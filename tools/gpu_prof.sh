#!/usr/bin/env bash
# ncu evidence: launch list of a bench step + full captures of the top kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export QLRT_NO_TORCH_PROFILER=1
NCU=ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench.log 2>&1
for spec in "gemm_fwd:gemm_kernel" "dequant:dequant64" "quantize:quantize64" "gemv:gemm_kernel"; do
  drv=${spec%%:*}; kre=${spec##*:}
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 \
    -o gpurun_out/prof_$drv -f python tools/prof_driver.py $drv > gpurun_out/ncu_$drv.log 2>&1
done
ls -la gpurun_out
