#!/usr/bin/env bash
# Build the sm_100a CUDA library in-tree: paper_2305_14314_b200/_lib/libqlrt_b200.so
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="$ROOT/paper_2305_14314_b200/csrc"
OUT="$ROOT/paper_2305_14314_b200/_lib"
mkdir -p "$OUT"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$ROOT/include -I$SRC ${QLRT_NVCC_EXTRA:-}"
objs=()
pids=()
for f in quant_kernels gemm_sm100 gemv_nf4 optim_kernels glue_kernels; do
  "$NVCC" $FLAGS -c "$SRC/$f.cu" -o "$OUT/$f${QLRT_LIB_NAME:+.$QLRT_LIB_NAME}.o" &
  pids+=($!)
  objs+=("$OUT/$f${QLRT_LIB_NAME:+.$QLRT_LIB_NAME}.o")
done
for p in "${pids[@]}"; do wait "$p"; done  # a failed compile fails the build
"$NVCC" -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/${QLRT_LIB_NAME:-libqlrt_b200.so}" "${objs[@]}" -lcudart
rm -f "${objs[@]}"
echo "built $OUT/${QLRT_LIB_NAME:-libqlrt_b200.so}"
# torch custom-op layer (torch.ops.qlrt_b200.*) over the C ABI
TORCH_DIR=$(python -c "import os, torch; print(os.path.dirname(torch.__file__))" 2>/dev/null)
ABI=$(python -c "import torch; print(int(torch._C._GLIBCXX_USE_CXX11_ABI))" 2>/dev/null)
g++ -O2 -std=c++17 -fPIC -shared -D_GLIBCXX_USE_CXX11_ABI=$ABI -DTORCH_API_INCLUDE_EXTENSION_H \
  -I"$ROOT/include" -I"$TORCH_DIR/include" -I"$TORCH_DIR/include/torch/csrc/api/include" -I/usr/local/cuda/include \
  "$SRC/torch_ops.cpp" -o "$OUT/libqlrt_torch_ops.so" \
  -L"$OUT" -lqlrt_b200 -L"$TORCH_DIR/lib" -ltorch -ltorch_cpu -ltorch_cuda -lc10 -lc10_cuda \
  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$ORIGIN' -Wl,-rpath,"$TORCH_DIR/lib"
echo "built $OUT/libqlrt_torch_ops.so"
