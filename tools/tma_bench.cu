// TMA throughput microbenchmark (tools only): one CTA per SM streams a large
// bf16 matrix [rows][cols] through a ring of S stages, each stage = `nbox`
// 2-d boxes of [box_rows][box_cols] (128B swizzle), issued by one thread,
// consumed by nobody (the barrier wait is the only consumer).  Reports GB/s
// for box shapes / stage counts, to size the skinny-GEMM and GEMV pipelines.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2305_14314_b200/csrc -Iinclude \
//        tools/tma_bench.cu -o /tmp/tma_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "sm100_ptx.cuh"

using namespace qlrt;

__global__ void __launch_bounds__(128, 1) tma_stream(const __grid_constant__ CUtensorMap tm, int stages, int nbox,
                                                     int box_rows, int box_bytes, int rows, int cols_boxes,
                                                     int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int stage_bytes = nbox * box_rows * box_bytes;
  // this CTA's row band, walked box by box (row-major over (row block, col box))
  // as a GEMM operand walk: each box of a stage has its own row block (the
  // CTA's rows), all boxes advance along the columns (K) stage by stage
  const int row_blocks = rows / box_rows;
  int cb = 0;
  auto issue = [&](int s) {
    ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
    for (int b = 0; b < nbox; ++b) {
      const int rb = (blockIdx.x + b * gridDim.x) % row_blocks;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              ptx::smem_u32(smem + s * stage_bytes + b * box_rows * box_bytes)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(ptx::smem_u32(&full[s])), "r"(cb * (box_bytes / 2)),
          "r"(rb * box_rows)
          : "memory");
    }
    cb = (cb + 1) % cols_boxes;
  };
  for (int s = 0; s < stages; ++s) issue(s);
  uint32_t par = 0;
  int s = 0;
  for (int i = 0; i < iters; ++i) {
    ptx::mbar_wait(&full[s], par);
    if (i + stages < iters) issue(s);
    if (++s == stages) {
      s = 0;
      par ^= 1u;
    }
  }
  if (iters < 0) *sink = smem[0];
}

// the GEMV's stage walk: 16 consecutive rows x 1 KB (one strip) per stage,
// the next stage the next 16 rows; CTAs start at different row offsets
__global__ void __launch_bounds__(128, 1) tma_rows(const __grid_constant__ CUtensorMap tm, int stages, int dims3,
                                                   int rows, int stage_bytes, int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int r0 = (int)(((long long)blockIdx.x * rows / gridDim.x) / 16 * 16);
  const int strip = blockIdx.x % 8;
  auto issue = [&](int s) {
    ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
    if (dims3)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
              ptx::smem_u32(smem + s * stage_bytes)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(ptx::smem_u32(&full[s])), "r"(0), "r"(r0), "r"(strip * 8)
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              ptx::smem_u32(smem + s * stage_bytes)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(ptx::smem_u32(&full[s])), "r"(strip * 256), "r"(r0)
          : "memory");
    r0 += 16;
    if (r0 >= rows) r0 = 0;
  };
  for (int s = 0; s < stages; ++s) issue(s);
  uint32_t par = 0;
  int s = 0;
  for (int i = 0; i < iters; ++i) {
    ptx::mbar_wait(&full[s], par);
    if (i + stages < iters) issue(s);
    if (++s == stages) {
      s = 0;
      par ^= 1u;
    }
  }
  if (iters < 0) *sink = smem[0];
}

// the GEMV's handshake: one producer warp (lane 0 issues) + `nc` consumer
// warps that wait on full[s] and arrive on empty[s]; the producer refills a
// slot once every consumer warp has arrived
__global__ void __launch_bounds__(544, 1) tma_rows_hs(const __grid_constant__ CUtensorMap tm, int stages, int nc,
                                                      int rows, int stage_bytes, int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], nc);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (warp == nc) {
    if (lane != 0) return;
    int r0 = (int)(((long long)blockIdx.x * rows / gridDim.x) / 16 * 16);
    const int strip = blockIdx.x % 8;
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      if (i >= stages) ptx::mbar_wait(&empty[s], (uint32_t)((i / stages) - 1) & 1u);
      ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
              ptx::smem_u32(smem + s * stage_bytes)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(ptx::smem_u32(&full[s])), "r"(0), "r"(r0), "r"(strip * 8)
          : "memory");
      r0 += 16;
      if (r0 >= rows) r0 = 0;
    }
    return;
  }
  if (warp > nc) return;
  uint32_t par = 0;
  int s = 0;
  for (int i = 0; i < iters; ++i) {
    ptx::mbar_wait(&full[s], par);
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
    if (++s == stages) {
      s = 0;
      par ^= 1u;
    }
  }
  if (iters < 0) *sink = smem[0];
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 16384, cols = 16384;  // 512 MB bf16 (> L2)
  void* buf;
  cudaMalloc(&buf, (size_t)rows * cols * 2);
  cudaMemset(buf, 1, (size_t)rows * cols * 2);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int shapes[][4] = {  // box_rows, box_bytes, nbox, stages
      {128, 128, 1, 4}, {128, 128, 1, 8}, {128, 128, 2, 4}, {128, 128, 2, 6}, {256, 128, 1, 4},
      {256, 128, 1, 6}, {64, 128, 1, 8},  {64, 128, 4, 4},  {32, 128, 8, 4},  {16, 128, 8, 8},
      {128, 64, 2, 8},  {256, 128, 2, 3}};
  for (auto& sh : shapes) {
    const int br = sh[0], bb = sh[1], nb = sh[2], st = sh[3];
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)(bb / 2), (cuuint32_t)br};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            bb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed\n");
      continue;
    }
    const int stage_bytes = nb * br * bb;
    const int iters = (int)((256ll << 20) / stage_bytes / sms);  // ~256 MB total
    const int smem = st * stage_bytes;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      tma_stream<<<sms, 128, smem>>>(tm, st, nb, br, bb, rows, cols * 2 / bb, iters, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)iters * stage_bytes * sms;
    printf("box %3d x %3d B, %d boxes/stage, %d stages (%3d KB in flight): %7.1f GB/s chip, %5.1f GB/s/SM  %s\n", br,
           bb, nb, st, smem / 1024, bytes / ms / 1e6, bytes / ms / 1e6 / sms, cudaGetErrorString(cudaGetLastError()));
  }
  // GEMV-like: rows of 8192 B (N = 16384 codes), 16 rows x 1 KB per stage
  {
    const int grows = 32768, row_bytes = 8192;  // 256 MB
    cudaFuncSetAttribute(tma_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int variant = 0; variant < 4; ++variant) {
      CUtensorMap tm;
      CUresult e;
      const bool d3 = variant < 2;
      const CUtensorMapL2promotion prom = (variant & 1) ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
      if (d3) {
        cuuint64_t dims[3] = {128, (cuuint64_t)grows, (cuuint64_t)(row_bytes / 128)};
        cuuint64_t strides[2] = {(cuuint64_t)row_bytes, 128};
        cuuint32_t box[3] = {128, 16, 8};
        cuuint32_t es[3] = {1, 1, 1};
        e = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        cuuint64_t dims[2] = {(cuuint64_t)(row_bytes / 4), (cuuint64_t)grows};
        cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
        cuuint32_t box[2] = {256, 16};
        cuuint32_t es[2] = {1, 1};
        e = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (e != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)e);
        continue;
      }
      for (int st : {4, 8, 12}) {
        const int stage_bytes = 16 * 1024;
        const int iters = (int)((256ll << 20) / stage_bytes / sms);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(a);
          tma_rows<<<sms, 128, st * stage_bytes>>>(tm, st, d3 ? 1 : 0, grows, stage_bytes, iters, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)iters * stage_bytes * sms;
        printf("gemv-like %s %s, %2d stages: %7.1f GB/s chip, %5.1f GB/s/SM %s\n", d3 ? "3d [8][16][128B] swz128" :
               "2d [16][1KB] u32 noswz", (variant & 1) ? "promo none " : "promo 256B", st, bytes / ms / 1e6,
               bytes / ms / 1e6 / sms, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  // the handshake variant (3-d box, 256B promotion)
  {
    const int grows = 32768, row_bytes = 8192;
    cudaFuncSetAttribute(tma_rows_hs, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    CUtensorMap tm;
    cuuint64_t dims[3] = {128, (cuuint64_t)grows, (cuuint64_t)(row_bytes / 128)};
    cuuint64_t strides[2] = {(cuuint64_t)row_bytes, 128};
    cuuint32_t box[3] = {128, 16, 8};
    cuuint32_t es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int nc : {1, 4, 16}) {
      for (int st : {8, 12}) {
        const int stage_bytes = 16 * 1024;
        const int iters = (int)((256ll << 20) / stage_bytes / sms);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(a);
          tma_rows_hs<<<sms, (nc + 1) * 32, st * stage_bytes>>>(tm, st, nc, grows, stage_bytes, iters, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)iters * stage_bytes * sms;
        printf("handshake: %2d consumer warps, %2d stages: %7.1f GB/s chip %s\n", nc, st, bytes / ms / 1e6,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
