#!/usr/bin/env bash
# full ncu capture of selected drivers: PROF="gemm_fwd:gemm_kernel dequant:dequant64"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in ${PROF:-gemm_fwd:gemm_kernel}; do
  drv=${spec%%:*}; kre=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kre -s ${SKIP:-2} -c 1 \
    -o gpurun_out/prof_$drv -f python tools/prof_driver.py $drv > gpurun_out/ncu_$drv.log 2>&1
  echo "$drv exit $?"
done
