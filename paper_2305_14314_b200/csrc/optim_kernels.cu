// Optimizer-side kernels: bit-exact fp32 Adam (reference AdamOptimizer.step,
// pkg/src/qlrt/training.py:426-442), the fp64 sum of squares and in-place
// scale of clip_global_norm (training.py:398-413), and the unified-memory
// prefetch that backs the paged moment store (paging.py's Pager, B200-native).
#include "qlrt_common.cuh"

namespace qlrt {

// One element, in the reference's op order with IEEE round-to-nearest on
// every step and no FMA contraction:
//   m *= b1; m += (1-b1)*g; v *= b2; v += (1-b2)*(g*g);
//   step = (m/bc1) / (sqrt(v/bc2) + eps); p -= lr*step
__device__ __forceinline__ void adam_one(float& p, float g, float& m, float& v, float b1, float omb1, float b2,
                                         float omb2, float bc1, float bc2, float eps, float lr) {
  m = __fmul_rn(m, b1);
  m = __fadd_rn(m, __fmul_rn(omb1, g));
  v = __fmul_rn(v, b2);
  v = __fadd_rn(v, __fmul_rn(omb2, __fmul_rn(g, g)));
  const float step = __fdiv_rn(__fdiv_rn(m, bc1), __fadd_rn(__fsqrt_rn(__fdiv_rn(v, bc2)), eps));
  p = __fsub_rn(p, __fmul_rn(lr, step));
}

__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                                                   float* __restrict__ m, float* __restrict__ v, int64_t n, float b1,
                                                   float omb1, float b2, float omb2, float bc1, float bc2, float eps,
                                                   float lr, __nv_bfloat16* __restrict__ pb) {
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool vec = ((((uintptr_t)p) | ((uintptr_t)g) | ((uintptr_t)m) | ((uintptr_t)v)) & 15) == 0 &&
                   (!pb || (((uintptr_t)pb) & 7) == 0);
  int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    for (int64_t i = i0; i < n4; i += stride) {
      float4 P = reinterpret_cast<float4*>(p)[i];
      const float4 G = reinterpret_cast<const float4*>(g)[i];
      float4 Mv = reinterpret_cast<float4*>(m)[i];
      float4 Vv = reinterpret_cast<float4*>(v)[i];
      adam_one(P.x, G.x, Mv.x, Vv.x, b1, omb1, b2, omb2, bc1, bc2, eps, lr);
      adam_one(P.y, G.y, Mv.y, Vv.y, b1, omb1, b2, omb2, bc1, bc2, eps, lr);
      adam_one(P.z, G.z, Mv.z, Vv.z, b1, omb1, b2, omb2, bc1, bc2, eps, lr);
      adam_one(P.w, G.w, Mv.w, Vv.w, b1, omb1, b2, omb2, bc1, bc2, eps, lr);
      reinterpret_cast<float4*>(p)[i] = P;
      reinterpret_cast<float4*>(m)[i] = Mv;
      reinterpret_cast<float4*>(v)[i] = Vv;
      if (pb) reinterpret_cast<uint2*>(pb)[i] = make_uint2(pack_bf16x2(P.x, P.y), pack_bf16x2(P.z, P.w));
    }
    for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      float P = p[i], Mv = m[i], Vv = v[i];
      adam_one(P, g[i], Mv, Vv, b1, omb1, b2, omb2, bc1, bc2, eps, lr);
      p[i] = P; m[i] = Mv; v[i] = Vv;
      if (pb) pb[i] = __float2bfloat16_rn(P);
    }
  } else {
    for (int64_t i = i0; i < n; i += stride) {
      float P = p[i], Mv = m[i], Vv = v[i];
      adam_one(P, g[i], Mv, Vv, b1, omb1, b2, omb2, bc1, bc2, eps, lr);
      p[i] = P; m[i] = Mv; v[i] = Vv;
      if (pb) pb[i] = __float2bfloat16_rn(P);
    }
  }
}

// Graph-replayable Adam over one flat parameter buffer: the step-dependent
// scalars come from device memory (hyper = b1, 1-b1, b2, 1-b2, bc1, bc2, eps,
// lr) and, with sumsq != nullptr, the global-norm clip is fused in
// (clip_global_norm, training.py:398-413: scale = f32(max_norm / sqrt(sumsq))
// when the norm exceeds max_norm, then g * scale in fp32 before the update).
__global__ void __launch_bounds__(256) adam_dev_kernel(float* __restrict__ p, const float* __restrict__ g,
                                                       float* __restrict__ m, float* __restrict__ v, int64_t n,
                                                       const float* __restrict__ hyper,
                                                       const double* __restrict__ sumsq, double max_norm,
                                                       __nv_bfloat16* __restrict__ pb) {
  const float b1 = hyper[0], omb1 = hyper[1], b2 = hyper[2], omb2 = hyper[3];
  const float bc1 = hyper[4], bc2 = hyper[5], eps = hyper[6], lr = hyper[7];
  float scale = 1.0f;
  bool clip = false;
  if (sumsq) {
    const double norm = __dsqrt_rn(*sumsq);
    if (norm > max_norm && norm > 0.0) {
      clip = true;
      scale = __double2float_rn(__ddiv_rn(max_norm, norm));
    }
  }
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 P = reinterpret_cast<float4*>(p)[i];
    float4 G = reinterpret_cast<const float4*>(g)[i];
    float4 Mv = reinterpret_cast<float4*>(m)[i];
    float4 Vv = reinterpret_cast<float4*>(v)[i];
    if (clip) {
      G.x = __fmul_rn(G.x, scale); G.y = __fmul_rn(G.y, scale);
      G.z = __fmul_rn(G.z, scale); G.w = __fmul_rn(G.w, scale);
    }
    adam_one(P.x, G.x, Mv.x, Vv.x, b1, omb1, b2, omb2, bc1, bc2, eps, lr);
    adam_one(P.y, G.y, Mv.y, Vv.y, b1, omb1, b2, omb2, bc1, bc2, eps, lr);
    adam_one(P.z, G.z, Mv.z, Vv.z, b1, omb1, b2, omb2, bc1, bc2, eps, lr);
    adam_one(P.w, G.w, Mv.w, Vv.w, b1, omb1, b2, omb2, bc1, bc2, eps, lr);
    reinterpret_cast<float4*>(p)[i] = P;
    reinterpret_cast<float4*>(m)[i] = Mv;
    reinterpret_cast<float4*>(v)[i] = Vv;
    if (pb) reinterpret_cast<uint2*>(pb)[i] = make_uint2(pack_bf16x2(P.x, P.y), pack_bf16x2(P.z, P.w));
  }
  for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float P = p[i], Mv = m[i], Vv = v[i], G = g[i];
    if (clip) G = __fmul_rn(G, scale);
    adam_one(P, G, Mv, Vv, b1, omb1, b2, omb2, bc1, bc2, eps, lr);
    p[i] = P; m[i] = Mv; v[i] = Vv;
    if (pb) pb[i] = __float2bfloat16_rn(P);
  }
}

// fp64 sum of squares: per-thread chains over a grid-stride range, then
// a fixed-shape tree per CTA and a fixed-order add of CTA partials by the
// last CTA (deterministic for a given n and grid).
__global__ void __launch_bounds__(256) sumsq_kernel(const float* __restrict__ g, int64_t n,
                                                    double* __restrict__ partials, unsigned* __restrict__ counter,
                                                    double* __restrict__ acc) {
  __shared__ double red[256];
  __shared__ bool last;
  // 16-byte loads, 8 in flight per thread, four independent fp64 chains
  // (x, y, z, w lanes of the float4s); the scalar tail goes to thread 0 of
  // CTA 0 -- a fixed order for a given n and grid
  // (a head of < 4 floats up to the first 16-byte boundary joins the tail)
  int64_t h = (int64_t)(((16u - (uint32_t)((uintptr_t)g & 15u)) & 15u) >> 2);
  h = h < n ? h : n;
  const float4* g4 = reinterpret_cast<const float4*>(g + h);
  const int64_t n4 = (n - h) >> 2, stride = (int64_t)gridDim.x * blockDim.x;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  auto add4 = [&](const float4 v) {
    s0 = __dadd_rn(s0, __dmul_rn((double)v.x, (double)v.x));
    s1 = __dadd_rn(s1, __dmul_rn((double)v.y, (double)v.y));
    s2 = __dadd_rn(s2, __dmul_rn((double)v.z, (double)v.z));
    s3 = __dadd_rn(s3, __dmul_rn((double)v.w, (double)v.w));
  };
  for (; j + 7 * stride < n4; j += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(g4 + j + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) add4(v[u]);
  }
  for (; j < n4; j += stride) add4(__ldg(g4 + j));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int64_t i = 0; i < h; ++i) s0 = __dadd_rn(s0, __dmul_rn((double)g[i], (double)g[i]));
    for (int64_t i = h + n4 * 4; i < n; ++i) s0 = __dadd_rn(s0, __dmul_rn((double)g[i], (double)g[i]));
  }
  red[threadIdx.x] = __dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3));
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = red[0];
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double t = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) t = __dadd_rn(t, ((volatile double*)partials)[b]);
    *acc = __dadd_rn(*acc, t);
    *counter = 0u;
  }
}

// numpy's pairwise sum of the float64 squares of one float32 tensor
// (np.sum(np.square(g, dtype=float64)), loops_utils.h.src pairwise_sum): the
// leaves (<= 128 values: 8 strided accumulators, combined
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail; < 8 values: sequential)
// in parallel, then the tree's internal nodes level by level in one CTA.
// The tree depends on n only; the host builds it (training.py).
__global__ void pairwise_leaves_kernel(const float* __restrict__ g, const int* __restrict__ leaves, int n_leaves,
                                       double* __restrict__ vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_leaves) return;
  const float* a = g + leaves[2 * i];
  const int n = leaves[2 * i + 1];
  double res;
  if (n < 8) {
    res = 0.0;
    for (int k = 0; k < n; ++k) res = __dadd_rn(res, __dmul_rn((double)a[k], (double)a[k]));
  } else {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dmul_rn((double)a[j], (double)a[j]);
    const int m = n - n % 8;
    for (int k = 8; k < m; k += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __dmul_rn((double)a[k + j], (double)a[k + j]));
    }
    res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                    __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (int k = m; k < n; ++k) res = __dadd_rn(res, __dmul_rn((double)a[k], (double)a[k]));
  }
  vals[i] = res;
}

// ops[3 j .. 3 j + 2] = (dst, left, right), grouped by tree height
// (level_starts[h] .. level_starts[h + 1]); acc += vals[root]
__global__ void __launch_bounds__(1024) pairwise_combine_kernel(double* __restrict__ vals, const int* __restrict__ ops,
                                                                const int* __restrict__ level_starts, int n_levels,
                                                                int root, double* __restrict__ acc) {
  for (int h = 0; h < n_levels; ++h) {
    for (int j = level_starts[h] + threadIdx.x; j < level_starts[h + 1]; j += blockDim.x)
      vals[ops[3 * j]] = __dadd_rn(vals[ops[3 * j + 1]], vals[ops[3 * j + 2]]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *acc = __dadd_rn(*acc, vals[root]);
}

__global__ void scale_kernel(float* __restrict__ g, int64_t n, float scale) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    g[i] = __fmul_rn(g[i], scale);
}

}  // namespace qlrt

using namespace qlrt;

extern "C" {

qlrt_status qlrt_adam_step(float* p, const float* g, float* m, float* v, int64_t n, float b1, float omb1, float b2,
                           float omb2, float bc1, float bc2, float eps, float lr, void* p_bf16, void* stream) {
  if (!p || !g || !m || !v || n <= 0) return QLRT_ERR_ARG;
  int64_t blocks = (n / 4 + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  adam_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(p, g, m, v, n, b1, omb1, b2, omb2, bc1, bc2, eps, lr,
                                                            (__nv_bfloat16*)p_bf16);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_adam_step_dev(float* p, const float* g, float* m, float* v, int64_t n, const float* hyper,
                               const double* sumsq, double max_norm, void* p_bf16, void* stream) {
  if (!p || !g || !m || !v || !hyper || n <= 0) return QLRT_ERR_ARG;
  if (((((uintptr_t)p) | ((uintptr_t)g) | ((uintptr_t)m) | ((uintptr_t)v)) & 15) || (((uintptr_t)p_bf16) & 7))
    return QLRT_ERR_ARG;
  int64_t blocks = (n / 4 + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  adam_dev_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(p, g, m, v, n, hyper, sumsq, max_norm,
                                                                (__nv_bfloat16*)p_bf16);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

// acc must point to a device double; the scratch (partials + counter) lives
// right after it: caller passes a buffer of >= 8 + 8*148*2 + 8 bytes.
qlrt_status qlrt_sumsq_f64(const float* g, int64_t n, double* acc, void* stream) {
  if (!g || !acc || n <= 0 || (((uintptr_t)g) & 3)) return QLRT_ERR_ARG;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 296) blocks = 296;
  double* partials = acc + 1;
  unsigned* counter = reinterpret_cast<unsigned*>(acc + 1 + 296);
  sumsq_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(g, n, partials, counter, acc);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_sumsq_f64_pairwise(const float* g, const int* leaves, int n_leaves, const int* ops,
                                    const int* level_starts, int n_levels, int root, double* vals, double* acc,
                                    void* stream) {
  if (!g || !leaves || n_leaves < 1 || !vals || !acc || n_levels < 0 || (n_levels > 0 && (!ops || !level_starts)))
    return QLRT_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  pairwise_leaves_kernel<<<(n_leaves + 255) / 256, 256, 0, st>>>(g, leaves, n_leaves, vals);
  QLRT_CHECK_LAUNCH();
  pairwise_combine_kernel<<<1, 1024, 0, st>>>(vals, ops, level_starts, n_levels, root, acc);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_scale_f32(float* g, int64_t n, float scale, void* stream) {
  if (!g || n <= 0) return QLRT_ERR_ARG;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  scale_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(g, n, scale);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_prefetch(void* ptr, size_t bytes, int device, void* stream) {
  if (!ptr || !bytes) return QLRT_ERR_ARG;
  const int dst = device >= 0 ? device : cudaCpuDeviceId;
  if (device >= 0) cudaMemAdvise(ptr, bytes, cudaMemAdviseSetPreferredLocation, device);
  cudaError_t e = cudaMemPrefetchAsync(ptr, bytes, dst, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return QLRT_ERR_CUDA;
  }
  return QLRT_OK;
}

}  // extern "C"
