// Fused elementwise kernels of the LLaMA-shaped harness (llama.py): RMSNorm,
// SwiGLU and rotary embedding, forward and backward, bf16 in/out with fp32
// math, 16-byte vector accesses.  Not on the reference's path (qlrt has no
// transformer); they keep the glue between the fused NF4 linears from
// dominating the C3/C5 step.
#include "qlrt_common.cuh"

namespace qlrt {
namespace glue {

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.0f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// y = x * rsqrt(mean(x^2) + eps), one CTA per row (h % 8 == 0)
__global__ void __launch_bounds__(256) rmsnorm_fwd_kernel(const uint4* __restrict__ x, uint4* __restrict__ y,
                                                          float* __restrict__ rstd, int h8, float eps) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (no early trigger: a fused GEMM launched
  // behind us would park its 1-CTA-per-SM grid on the SMs we still need)
  __shared__ float red[8];
  const int64_t row = blockIdx.x;
  const uint4* xr = x + row * h8;
  float ss = 0.0f;
  for (int i = threadIdx.x; i < h8; i += blockDim.x) {
    const uint4 u = xr[i];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) ss += bf_lo(w[j]) * bf_lo(w[j]) + bf_hi(w[j]) * bf_hi(w[j]);
  }
  const float r = rsqrtf(block_sum(ss, red) / (float)(h8 * 8) + eps);
  if (threadIdx.x == 0) rstd[row] = r;
  uint4* yr = y + row * h8;
  for (int i = threadIdx.x; i < h8; i += blockDim.x) {
    const uint4 u = xr[i];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = pack_bf16x2(bf_lo(w[j]) * r, bf_hi(w[j]) * r);
    yr[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// s = x + d (the residual stream), y = s * rsqrt(mean(s^2) + eps): the
// residual add fused into the next norm (one read of x and d, s and y written)
__global__ void __launch_bounds__(256) add_rmsnorm_fwd_kernel(const uint4* __restrict__ x, const uint4* __restrict__ d,
                                                              uint4* __restrict__ s, uint4* __restrict__ y,
                                                              float* __restrict__ rstd, int h8, float eps) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (no early trigger: a fused GEMM launched
  // behind us would park its 1-CTA-per-SM grid on the SMs we still need)
  __shared__ float red[8];
  const int64_t row = blockIdx.x;
  const uint4 *xr = x + row * h8, *dr = d + row * h8;
  uint4* sr = s + row * h8;
  float ss = 0.0f;
  for (int i = threadIdx.x; i < h8; i += blockDim.x) {
    const uint4 a = xr[i], b = dr[i];
    const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // bf16(x + d) as torch's bf16 add rounds it, then the norm of the rounded sum
      o[j] = pack_bf16x2(bf_lo(wa[j]) + bf_lo(wb[j]), bf_hi(wa[j]) + bf_hi(wb[j]));
      ss += bf_lo(o[j]) * bf_lo(o[j]) + bf_hi(o[j]) * bf_hi(o[j]);
    }
    sr[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
  const float r = rsqrtf(block_sum(ss, red) / (float)(h8 * 8) + eps);
  if (threadIdx.x == 0) rstd[row] = r;
  uint4* yr = y + row * h8;
  for (int i = threadIdx.x; i < h8; i += blockDim.x) {
    const uint4 u = sr[i];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = pack_bf16x2(bf_lo(w[j]) * r, bf_hi(w[j]) * r);
    yr[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// dx = r * dy - r^3 * x * sum(dy * x) / h  (+ dres: the residual branch's gradient)
__global__ void __launch_bounds__(256) rmsnorm_bwd_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ x,
                                                          const float* __restrict__ rstd, uint4* __restrict__ dx,
                                                          int h8, const uint4* __restrict__ dres) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (no early trigger: a fused GEMM launched
  // behind us would park its 1-CTA-per-SM grid on the SMs we still need)
  __shared__ float red[8];
  const int64_t row = blockIdx.x;
  const uint4 *xr = x + row * h8, *gr = dy + row * h8;
  float dot = 0.0f;
  for (int i = threadIdx.x; i < h8; i += blockDim.x) {
    const uint4 a = xr[i], b = gr[i];
    const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) dot += bf_lo(wa[j]) * bf_lo(wb[j]) + bf_hi(wa[j]) * bf_hi(wb[j]);
  }
  dot = block_sum(dot, red);
  const float r = rstd[row];
  const float k = r * r * r * dot / (float)(h8 * 8);
  uint4* dr = dx + row * h8;
  for (int i = threadIdx.x; i < h8; i += blockDim.x) {
    const uint4 a = xr[i], b = gr[i];
    const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
    uint32_t o[4];
    if (dres) {  // + the residual gradient: d(x + delta) feeds both branches
      const uint4 c = dres[row * h8 + i];
      const uint32_t wc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        // bf16(rmsnorm grad) + dres, as the separate kernels + torch add round it
        const uint32_t g = pack_bf16x2(r * bf_lo(wb[j]) - k * bf_lo(wa[j]), r * bf_hi(wb[j]) - k * bf_hi(wa[j]));
        o[j] = pack_bf16x2(bf_lo(g) + bf_lo(wc[j]), bf_hi(g) + bf_hi(wc[j]));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        o[j] = pack_bf16x2(r * bf_lo(wb[j]) - k * bf_lo(wa[j]), r * bf_hi(wb[j]) - k * bf_hi(wa[j]));
    }
    dr[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__device__ __forceinline__ float sigmoidf_(float g) { return 1.0f / (1.0f + __expf(-g)); }

// out = silu(g) * u over rows x (c8 * 8) elements, row pitches in 16 B units
// (contiguous: one row; concatenated [g | u]: ldg = ldu = 2 c8)
__global__ void swiglu_fwd_kernel(const uint4* __restrict__ g, const uint4* __restrict__ u, uint4* __restrict__ out,
                                  int64_t rows, int64_t c8, int64_t ldg, int64_t ldu, int64_t ldo) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (no early trigger: a fused GEMM launched
  // behind us would park its 1-CTA-per-SM grid on the SMs we still need)
  // rows on grid y, 16-byte columns on grid x (no 64-bit divisions on the element path)
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < c8; c += (int64_t)gridDim.x * blockDim.x) {
    const uint4 a = g[r * ldg + c], b = u[r * ldu + c];
    const int64_t i = r * ldo + c;
    const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float g0 = bf_lo(wa[j]), g1 = bf_hi(wa[j]);
      o[j] = pack_bf16x2(g0 * sigmoidf_(g0) * bf_lo(wb[j]), g1 * sigmoidf_(g1) * bf_hi(wb[j]));
    }
    out[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// du = dout * silu(g);  dg = dout * u * s * (1 + g (1 - s)),  s = sigmoid(g)
__global__ void swiglu_bwd_kernel(const uint4* __restrict__ g, const uint4* __restrict__ u,
                                  const uint4* __restrict__ dout, uint4* __restrict__ dg, uint4* __restrict__ du,
                                  int64_t rows, int64_t c8, int64_t ldgu, int64_t ldo) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (no early trigger: a fused GEMM launched
  // behind us would park its 1-CTA-per-SM grid on the SMs we still need)
  // rows on grid y, 16-byte columns on grid x (no 64-bit divisions on the element path)
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
  for (int64_t cc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; cc < c8; cc += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = r * ldgu + cc;  // g, u, dg, du share a pitch
    const uint4 a = g[i], b = u[i], c = dout[r * ldo + cc];
    const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w}, wc[4] = {c.x, c.y, c.z, c.w};
    uint32_t og[4], ou[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float gg[2] = {bf_lo(wa[j]), bf_hi(wa[j])}, uu[2] = {bf_lo(wb[j]), bf_hi(wb[j])};
      float dd[2] = {bf_lo(wc[j]), bf_hi(wc[j])}, rg[2], ru[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float s = sigmoidf_(gg[e]);
        ru[e] = dd[e] * gg[e] * s;
        rg[e] = dd[e] * uu[e] * s * (1.0f + gg[e] * (1.0f - s));
      }
      og[j] = pack_bf16x2(rg[0], rg[1]);
      ou[j] = pack_bf16x2(ru[0], ru[1]);
    }
    dg[i] = make_uint4(og[0], og[1], og[2], og[3]);
    du[i] = make_uint4(ou[0], ou[1], ou[2], ou[3]);
  }
}

// rotary embedding on [rows = b*s, heads, d] bf16, adjacent pairs (2i, 2i+1)
// rotated by angle pos * inv_freq[i]; cs = (cos, sin) fp32 [s][d/2]; sign = -1
// applies the inverse rotation (backward)
// (row pitches ldx / ldy in 16 B units: q or k read from / written to a
// column slice of the concatenated q | k | v projection)
__global__ void rope_kernel(const uint4* __restrict__ x, uint4* __restrict__ y, const float2* __restrict__ cs,
                            int64_t rows, int heads, int d, int seq, float sign, int64_t ldx, int64_t ldy) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (no early trigger: a fused GEMM launched
  // behind us would park its 1-CTA-per-SM grid on the SMs we still need)
  const int d8 = d / 8;
  const int rw = d8 * heads;
  // one CTA per row: the position once, 32-bit column arithmetic
  const int64_t row = blockIdx.x;
  const int pos = (int)(row % seq);
  for (int within = threadIdx.x; within < rw; within += blockDim.x) {
    const int c8 = within % d8;
    const float2* t = cs + (int64_t)pos * (d / 2) + c8 * 4;  // 4 pairs per 16 B
    const int64_t i = row * ldy + within;
    const uint4 a = x[row * ldx + within];
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 r = t[j];
      const float x0 = bf_lo(w[j]), x1 = bf_hi(w[j]), sn = sign * r.y;
      o[j] = pack_bf16x2(x0 * r.x - x1 * sn, x0 * sn + x1 * r.x);
    }
    y[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// q | k | v rows of the concatenated projection <-> separate q, k, v (rows x
// h, h = heads * d): forward rotates q and k and copies v out of ycat;
// backward (sign = -1) writes the inverse-rotated dq, dk and dv into dycat
template <bool FWD>
__global__ void rope_qkv_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b, const uint4* __restrict__ c,
                                uint4* __restrict__ x, uint4* __restrict__ y, uint4* __restrict__ z,
                                const float2* __restrict__ cs, int64_t rows, int h8, int d, int seq) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (no early trigger: a fused GEMM launched
  // behind us would park its 1-CTA-per-SM grid on the SMs we still need)
  // FWD: a = ycat (rows x 3 h8), x / y / z = q / k / v;  BWD: a / b / c = dq / dk / dv, x = dycat
  const int d8 = d / 8;
  // one CTA per row: the position once, the q / k / v parts as an outer loop
  const int64_t row = blockIdx.x;
  const int pos = (int)(row % seq);
  for (int part = 0; part < 3; ++part)
  for (int e = threadIdx.x; e < h8; e += blockDim.x) {
    const int64_t k = row * 3 * h8 + (int64_t)part * h8 + e;
    uint4 v;
    if (FWD) v = a[k];
    else v = (part == 0 ? a : part == 1 ? b : c)[row * h8 + e];
    if (part < 2) {
      const int c8 = e % d8;
      const float2* t = cs + (int64_t)pos * (d / 2) + c8 * 4;
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 r = t[j];
        const float x0 = bf_lo(wv[j]), x1 = bf_hi(wv[j]), sn = FWD ? r.y : -r.y;
        o[j] = pack_bf16x2(x0 * r.x - x1 * sn, x0 * sn + x1 * r.x);
      }
      v = make_uint4(o[0], o[1], o[2], o[3]);
    }
    if (FWD) (part == 0 ? x : part == 1 ? y : z)[row * h8 + e] = v;
    else x[k] = v;
  }
}

// cross entropy over bf16 logit rows (the harness's loss; torch computes it
// in fp32 from a materialized fp32 copy of the logits): one CTA per row,
// online max / sum-exp in one pass, loss[row] = lse - x[target]
__global__ void __launch_bounds__(256) xent_fwd_kernel(const uint4* __restrict__ logits, const int64_t* __restrict__ tgt,
                                                       int v8, float* __restrict__ loss, float* __restrict__ lse_out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (no early trigger: a fused GEMM launched
  // behind us would park its 1-CTA-per-SM grid on the SMs we still need)
  __shared__ float sm[8], ss[8];
  const int64_t row = blockIdx.x;
  const uint4* x = logits + row * v8;
  float m = -INFINITY, sum = 0.0f;
  for (int i = threadIdx.x; i < v8; i += blockDim.x) {
    const uint4 u = x[i];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    float e[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      e[2 * j] = bf_lo(w[j]);
      e[2 * j + 1] = bf_hi(w[j]);
    }
    float bm = e[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) bm = fmaxf(bm, e[j]);
    const float nm = fmaxf(m, bm);
    float acc = sum * __expf(m - nm);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += __expf(e[j] - nm);
    m = nm;
    sum = acc;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, sum, o);
    const float nm = fmaxf(m, om);
    sum = (m == -INFINITY ? 0.0f : sum * __expf(m - nm)) + (om == -INFINITY ? 0.0f : os * __expf(om - nm));
    m = nm;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sm[w] = m;
    ss[w] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm[0], S = ss[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
      const float nm = fmaxf(M, sm[i]);
      S = S * __expf(M - nm) + ss[i] * __expf(sm[i] - nm);
      M = nm;
    }
    const float lse = M + logf(S);
    const int64_t t = tgt[row];
    const unsigned short xb = reinterpret_cast<const unsigned short*>(x)[t];
    loss[row] = lse - __uint_as_float((uint32_t)xb << 16);
    lse_out[row] = lse;
  }
}
// d logits[row][v] = (softmax - onehot(target)) * g / rows   (bf16 out)
__global__ void xent_bwd_kernel(const uint4* __restrict__ logits, const int64_t* __restrict__ tgt,
                                const float* __restrict__ lse, const float* __restrict__ grad, int v8, float inv_rows,
                                uint4* __restrict__ dlogits) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (no early trigger: a fused GEMM launched
  // behind us would park its 1-CTA-per-SM grid on the SMs we still need)
  const int64_t row = blockIdx.x;
  const float L = lse[row], sc = *grad * inv_rows;
  const int64_t t = tgt[row];
  const uint4* x = logits + row * v8;
  uint4* d = dlogits + row * v8;
  for (int i = threadIdx.x; i < v8; i += blockDim.x) {
    const uint4 u = x[i];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t v0 = (int64_t)i * 8 + 2 * j;
      const float p0 = __expf(bf_lo(w[j]) - L) - (v0 == t ? 1.0f : 0.0f);
      const float p1 = __expf(bf_hi(w[j]) - L) - (v0 + 1 == t ? 1.0f : 0.0f);
      o[j] = pack_bf16x2(p0 * sc, p1 * sc);
    }
    d[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// programmatic dependent launch: the glue kernel may be scheduled while its
// predecessor (a fused GEMM) drains; it waits before touching memory
template <typename... KArgs, typename... Args>
static qlrt_status launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = policy(P_PDL) ? 1 : 0;
  if (policy(P_PRIO) == 1) {  // (the step's critical path: ahead of side-stream work)
    at[cfg.numAttrs].id = cudaLaunchAttributePriority;
    at[cfg.numAttrs].val.priority = high_priority();
    cfg.numAttrs += 1;
  }
  if (cudaLaunchKernelEx(&cfg, k, ((KArgs)args)...) != cudaSuccess) return QLRT_ERR_CUDA;
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

// (columns, rows) grid of an elementwise row kernel: 256-thread column blocks
static dim3 grid_rows(int64_t rows, int64_t c8) {
  const int64_t gx = (c8 + 255) / 256, gy = rows;
  const int64_t cx = gx < (int64_t)kNumSMs * 8 ? gx : (int64_t)kNumSMs * 8;
  return dim3((unsigned)(cx < 1 ? 1 : cx), (unsigned)(gy < 65535 ? gy : 65535));
}

}  // namespace glue
}  // namespace qlrt

using namespace qlrt;

extern "C" {

qlrt_status qlrt_rmsnorm_fwd(const void* x, void* y, float* rstd, int64_t rows, int64_t h, float eps, void* stream) {
  if (!x || !y || !rstd || rows <= 0 || h <= 0 || (h % 8)) return QLRT_ERR_ARG;
  return glue::launch_pdl(glue::rmsnorm_fwd_kernel, dim3((unsigned)rows), dim3(256), (cudaStream_t)stream,
                          (const uint4*)x, (uint4*)y, rstd,
                                                                            (int)(h / 8), eps);
}

qlrt_status qlrt_rmsnorm_bwd(const void* dy, const void* x, const float* rstd, void* dx, int64_t rows, int64_t h,
                             void* stream) {
  if (!dy || !x || !rstd || !dx || rows <= 0 || h <= 0 || (h % 8)) return QLRT_ERR_ARG;
  return glue::launch_pdl(glue::rmsnorm_bwd_kernel, dim3((unsigned)rows), dim3(256), (cudaStream_t)stream,
                          (const uint4*)dy, (const uint4*)x, rstd,
                                                                            (uint4*)dx, (int)(h / 8), nullptr);
}
qlrt_status qlrt_add_rmsnorm_fwd(const void* x, const void* d, void* s, void* y, float* rstd, int64_t rows, int64_t h,
                                 float eps, void* stream) {
  if (!x || !d || !s || !y || !rstd || rows <= 0 || h <= 0 || (h % 8)) return QLRT_ERR_ARG;
  return glue::launch_pdl(glue::add_rmsnorm_fwd_kernel, dim3((unsigned)rows), dim3(256), (cudaStream_t)stream,
                          (const uint4*)x, (const uint4*)d, (uint4*)s, (uint4*)y, rstd, (int)(h / 8), eps);
}
qlrt_status qlrt_rmsnorm_bwd_add(const void* dy, const void* x, const float* rstd, const void* dres, void* dx,
                                 int64_t rows, int64_t h, void* stream) {
  if (!dy || !x || !rstd || !dres || !dx || rows <= 0 || h <= 0 || (h % 8)) return QLRT_ERR_ARG;
  return glue::launch_pdl(glue::rmsnorm_bwd_kernel, dim3((unsigned)rows), dim3(256), (cudaStream_t)stream,
                          (const uint4*)dy, (const uint4*)x, rstd, (uint4*)dx, (int)(h / 8), (const uint4*)dres);
}

qlrt_status qlrt_swiglu_fwd(const void* g, const void* u, void* out, int64_t n, void* stream) {
  if (!g || !u || !out || n <= 0 || (n % 8)) return QLRT_ERR_ARG;
  return glue::launch_pdl(glue::swiglu_fwd_kernel, glue::grid_rows(1, n / 8), dim3(256), (cudaStream_t)stream,
                          (const uint4*)g, (const uint4*)u, (uint4*)out, 1, n / 8, 0, 0, 0);
}

qlrt_status qlrt_swiglu_bwd(const void* g, const void* u, const void* dout, void* dg, void* du, int64_t n,
                            void* stream) {
  if (!g || !u || !dout || !dg || !du || n <= 0 || (n % 8)) return QLRT_ERR_ARG;
  return glue::launch_pdl(glue::swiglu_bwd_kernel, glue::grid_rows(1, n / 8), dim3(256), (cudaStream_t)stream,
                          (const uint4*)g, (const uint4*)u, (const uint4*)dout, (uint4*)dg, (uint4*)du, 1, n / 8, 0, 0);
}

qlrt_status qlrt_rope(const void* x, void* y, const void* cos_sin, int64_t rows, int heads, int d, int seq,
                      int inverse, void* stream) {
  if (!x || !y || !cos_sin || rows <= 0 || heads <= 0 || d <= 0 || (d % 8) || seq <= 0) return QLRT_ERR_ARG;
  const int64_t rw = (int64_t)heads * (d / 8);
  return glue::launch_pdl(glue::rope_kernel, dim3((unsigned)rows), dim3(256), (cudaStream_t)stream,
                          (const uint4*)x, (uint4*)y, (const float2*)cos_sin, rows, heads, d, seq, inverse ? -1.0f : 1.0f, rw, rw);
}
qlrt_status qlrt_rope_strided(const void* x, int64_t ldx, void* y, int64_t ldy, const void* cos_sin, int64_t rows,
                              int heads, int d, int seq, int inverse, void* stream) {
  if (!x || !y || !cos_sin || rows <= 0 || heads <= 0 || d <= 0 || (d % 8) || seq <= 0 || (ldx % 8) || (ldy % 8) ||
      ldx < (int64_t)heads * d || ldy < (int64_t)heads * d)
    return QLRT_ERR_ARG;
  return glue::launch_pdl(glue::rope_kernel, dim3((unsigned)rows), dim3(256), (cudaStream_t)stream,
                          (const uint4*)x, (uint4*)y, (const float2*)cos_sin, rows, heads, d, seq, inverse ? -1.0f : 1.0f, ldx / 8,
      ldy / 8);
}
qlrt_status qlrt_rope_qkv_fwd(const void* ycat, void* q, void* k, void* v, const void* cos_sin, int64_t rows,
                              int heads, int d, int seq, void* stream) {
  if (!ycat || !q || !k || !v || !cos_sin || rows <= 0 || heads <= 0 || d <= 0 || (d % 8) || seq <= 0)
    return QLRT_ERR_ARG;
  const int h8 = heads * d / 8;
  return glue::launch_pdl(glue::rope_qkv_kernel<true>, dim3((unsigned)rows), dim3(256), (cudaStream_t)stream,
                          (const uint4*)ycat, nullptr, nullptr, (uint4*)q, (uint4*)k, (uint4*)v, (const float2*)cos_sin, rows, h8, d, seq);
}
qlrt_status qlrt_rope_qkv_bwd(const void* dq, const void* dk, const void* dv, void* dycat, const void* cos_sin,
                              int64_t rows, int heads, int d, int seq, void* stream) {
  if (!dq || !dk || !dv || !dycat || !cos_sin || rows <= 0 || heads <= 0 || d <= 0 || (d % 8) || seq <= 0)
    return QLRT_ERR_ARG;
  const int h8 = heads * d / 8;
  return glue::launch_pdl(glue::rope_qkv_kernel<false>, dim3((unsigned)rows), dim3(256), (cudaStream_t)stream,
                          (const uint4*)dq, (const uint4*)dk, (const uint4*)dv, (uint4*)dycat, nullptr, nullptr, (const float2*)cos_sin,
      rows, h8, d, seq);
}
qlrt_status qlrt_xent_fwd(const void* logits, const int64_t* targets, int64_t rows, int64_t vocab, float* loss,
                          float* lse, void* stream) {
  if (!logits || !targets || !loss || !lse || rows <= 0 || vocab <= 0 || (vocab % 8)) return QLRT_ERR_ARG;
  return glue::launch_pdl(glue::xent_fwd_kernel, dim3((unsigned)rows), dim3(256), (cudaStream_t)stream,
                          (const uint4*)logits, targets,
                                                                          (int)(vocab / 8), loss, lse);
}
qlrt_status qlrt_xent_bwd(const void* logits, const int64_t* targets, const float* lse, const float* grad,
                          int64_t rows, int64_t vocab, void* dlogits, void* stream) {
  if (!logits || !targets || !lse || !grad || !dlogits || rows <= 0 || vocab <= 0 || (vocab % 8)) return QLRT_ERR_ARG;
  return glue::launch_pdl(glue::xent_bwd_kernel, dim3((unsigned)rows), dim3(256), (cudaStream_t)stream,
                          (const uint4*)logits, targets, lse, grad, (int)(vocab / 8), 1.0f / (float)rows, (uint4*)dlogits);
}
// concatenated [g | u] rows (cols each): out[rows][cols] = silu(g) * u
qlrt_status qlrt_swiglu_cat_fwd(const void* gu, void* out, int64_t rows, int64_t cols, void* stream) {
  if (!gu || !out || rows <= 0 || cols <= 0 || (cols % 8)) return QLRT_ERR_ARG;
  const int64_t c8 = cols / 8;
  return glue::launch_pdl(glue::swiglu_fwd_kernel, glue::grid_rows(rows, c8), dim3(256), (cudaStream_t)stream,
                          (const uint4*)gu, (const uint4*)gu + c8, (uint4*)out, rows, c8, 2 * c8, 2 * c8, c8);
}
// d[g | u] rows from dout[rows][cols] and the saved [g | u]
qlrt_status qlrt_swiglu_cat_bwd(const void* gu, const void* dout, void* dgu, int64_t rows, int64_t cols,
                                void* stream) {
  if (!gu || !dout || !dgu || rows <= 0 || cols <= 0 || (cols % 8)) return QLRT_ERR_ARG;
  const int64_t c8 = cols / 8;
  return glue::launch_pdl(glue::swiglu_bwd_kernel, glue::grid_rows(rows, c8), dim3(256), (cudaStream_t)stream,
                          (const uint4*)gu, (const uint4*)gu + c8, (const uint4*)dout, (uint4*)dgu, (uint4*)dgu + c8, rows, c8, 2 * c8,
      c8);
}

}  // extern "C"
