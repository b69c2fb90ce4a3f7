// Batch-1 NF4 GEMV for sm_100a: y[N] = x[K] W + s (x l1) l2   (qlora.py:124-148 at M = 1).
//
// Reads the packed codes (0.5 B/weight + 1 DQ byte per 64) once; no tensor
// cores (one live column), no dequantized copy of W.  Each lane owns one
// 64-column block of a 2048-column strip and walks rows of W:
//   * one 256-bit load of the row's 32 code bytes (a warp reads 1 KB
//     contiguous), the DQ byte and c1 -> block constant c (exact fp64
//     dq_decompress arithmetic, doublequant.py:190-195), next row prefetched;
//   * a 16-entry bf16 table bf16(f32(v_q) * c) -- the same decode as the fused
//     GEMM producer;
//   * decode + FHFMA.BF16 (fp32 acc += bf16(w) * bf16(x_k), exact products):
//     words [0, WL) of the 8 per block look the table up in a per-lane
//     shared-memory column (one LOP3 + one LDS per code, bank = lane); words
//     [WL, 8) use register byte-permutes (lookup8, ~2 PRMT per code).  The mix
//     balances the ALU pipe against the shared-memory pipe: the kernel is
//     bound by decode instruction issue, not by HBM (GEMV).
// The 8 warps of a CTA split the CTA's rows and reduce through shared memory;
// CTAs split K, write fp32 partials, and the last CTA of a strip (atomic
// ticket) sums the partials in split order (deterministic), adds the LoRA
// term and writes bf16 y.
#include <stdlib.h>

#include "qlrt_common.cuh"

namespace qlrt {
namespace gemv {

constexpr int TPB = 256;
constexpr int WARPS = TPB / 32;
constexpr int STRIP = 32 * 64;  // columns per CTA
constexpr int SMS_X2 = 2 * kNumSMs;

struct Plan {
  int strips, zc, zt;
};

static Plan plan(int64_t K, int64_t N) {
  Plan p;
  p.strips = (int)cdiv(N, STRIP);
  int64_t zc = SMS_X2 / p.strips;
  if (zc < 1) zc = 1;
  if (zc > K / WARPS) zc = K / WARPS > 0 ? K / WARPS : 1;
  p.zc = (int)zc;
  p.zt = (int)cdiv(K, 128);
  return p;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// workspace: [partials zc*N f32][tpart zt*r f32][counters strips u32]
static size_t ws_bytes(int64_t K, int64_t N, int r) {
  const Plan p = plan(K, N);
  return align256((size_t)p.zc * N * 4) + align256((size_t)p.zt * (r > 0 ? r : 1) * 4) +
         align256((size_t)p.strips * 4);
}

__device__ __forceinline__ void ld_v8(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}

// 8 codes (nibbles of w, element order) -> 8 bf16 in o[0..3] from lo/hi byte planes
__device__ __forceinline__ void lookup8(uint32_t w, const uint32_t (&L)[4], const uint32_t (&H)[4], uint32_t (&o)[4]) {
  const uint32_t sel = w & 0x77777777u;
  const uint32_t bs = ((w >> 1) & 0x44444444u) | 0x32103210u;
  const uint32_t selh = sel >> 16, bsh = bs >> 16;
  const uint32_t la = __byte_perm(__byte_perm(L[0], L[1], sel), __byte_perm(L[2], L[3], sel), bs);
  const uint32_t ha = __byte_perm(__byte_perm(H[0], H[1], sel), __byte_perm(H[2], H[3], sel), bs);
  const uint32_t lb = __byte_perm(__byte_perm(L[0], L[1], selh), __byte_perm(L[2], L[3], selh), bsh);
  const uint32_t hb = __byte_perm(__byte_perm(H[0], H[1], selh), __byte_perm(H[2], H[3], selh), bsh);
  o[0] = __byte_perm(la, ha, 0x5140);
  o[1] = __byte_perm(la, ha, 0x7362);
  o[2] = __byte_perm(lb, hb, 0x5140);
  o[3] = __byte_perm(lb, hb, 0x7362);
}

// acc0 += bf16(lo half of w) * x, acc1 += bf16(hi half of w) * x  (FHFMA.BF16)
__device__ __forceinline__ void fma2_bf16(float& a0, float& a1, uint32_t w, unsigned short x) {
  asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
      "fma.rn.f32.bf16 %0, lo, %3, %0;\n\t"
      "fma.rn.f32.bf16 %1, hi, %3, %1;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "r"(w), "h"(x));
}

struct Vals32 {
  float v[16];
};

template <int WL>
__global__ void __launch_bounds__(TPB, 2)
    gemv_nf4_kernel(const uint8_t* __restrict__ codes, const uint8_t* __restrict__ dq_codes,
                    const float* __restrict__ c1, const float* __restrict__ mu, int bs2_shift, qlrt_fp8spec sp,
                    Vals32 vals, int64_t K, int64_t N, const unsigned short* __restrict__ x, float* __restrict__ part,
                    unsigned* __restrict__ counters, const float* __restrict__ tpart, int zt,
                    const __nv_bfloat16* __restrict__ l2, int rank, float s, __nv_bfloat16* __restrict__ y) {
  extern __shared__ __align__(16) float4 red[];  // [WARPS][32 lanes][16 float4], chunk-swizzled
  __shared__ double fp8_lut[256];
  __shared__ float tsh[512];
  __shared__ unsigned last_flag;
  // per-lane private copy of the row-block's table (bank = lane), 2 KB-aligned at run time
  __shared__ __align__(16) uint32_t tab_raw[WARPS * 16 * 32 + 512];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int strip = blockIdx.x, z = blockIdx.y, zc = gridDim.y;
  const int64_t nbr = N / 64;
  const int64_t jb = (int64_t)strip * 32 + lane;
  const bool live = jb < nbr;
  const int64_t r0 = K * z / zc, r1 = K * (z + 1) / zc;
  // byte address of this lane's table column; entry q at + q * 128
  const uint32_t tbase = ((((uint32_t)__cvta_generic_to_shared(tab_raw)) + 2047u) & ~2047u) + wid * 2048u + lane * 4u;

  uint32_t cw[8];
  uint32_t dqb = 0;
  float c1v = 0.0f;
  unsigned short xk = 0;
  auto fetch = [&](int64_t k) {
    const int64_t blk = k * nbr + jb;
    xk = __ldg(x + k);
    if (live) {
      ld_v8(codes + blk * 32, cw);
      dqb = __ldg(dq_codes + blk);
      c1v = __ldg(c1 + (blk >> bs2_shift));
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) cw[i] = 0u;
    }
  };
  int64_t k = r0 + wid;
  if (k < r1) fetch(k);
  fp8_lut[threadIdx.x] = fp8_decode_fast(threadIdx.x, sp);
  __syncthreads();
  const double mu_d = (double)__ldg(mu);

  float acc[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) acc[i] = 0.0f;
  for (; k < r1; k += WARPS) {
    uint32_t cur[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) cur[i] = cw[i];
    const unsigned short xc = xk;
    const double rr = __dadd_rn(__dmul_rn(fp8_lut[dqb], (double)c1v), mu_d);
    const float c = __double2float_rn(rr > 0.0 ? rr : 0.0);
    if (k + WARPS < r1) fetch(k + WARPS);
    uint32_t L[4], H[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t p0 = pack_bf16x2(vals.v[4 * q] * c, vals.v[4 * q + 1] * c);
      const uint32_t p1 = pack_bf16x2(vals.v[4 * q + 2] * c, vals.v[4 * q + 3] * c);
      L[q] = __byte_perm(p0, p1, 0x6420);
      H[q] = __byte_perm(p0, p1, 0x7531);
      if (WL > 0) {  // entry e in the low half of word e (FHFMA reads .H0)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(tbase + (4 * q) * 128), "r"(p0));
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(tbase + (4 * q + 1) * 128), "r"(__umulhi(p0, 0x10000u)));
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(tbase + (4 * q + 2) * 128), "r"(p1));
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(tbase + (4 * q + 3) * 128), "r"(__umulhi(p1, 0x10000u)));
      }
    }
    // words [0, WL): nibble -> table address (shift on the FMA pipe, one LOP3), LDS, FHFMA
#pragma unroll
    for (int wd = 0; wd < WL; ++wd) {
      const uint32_t w = cur[wd];
      uint32_t a[8];
      a[0] = ((w << 7) & 0x780u) | tbase;
      a[1] = ((w << 3) & 0x780u) | tbase;
      a[2] = (__umulhi(w, 0x80000000u) & 0x780u) | tbase;
      a[3] = (__umulhi(w, 0x8000000u) & 0x780u) | tbase;
      a[4] = (__umulhi(w, 0x800000u) & 0x780u) | tbase;
      a[5] = (__umulhi(w, 0x80000u) & 0x780u) | tbase;
      a[6] = (__umulhi(w, 0x8000u) & 0x780u) | tbase;
      a[7] = (__umulhi(w, 0x800u) & 0x780u) | tbase;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        uint32_t t;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(t) : "r"(a[e]));
        asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\t"
            "fma.rn.f32.bf16 %0, lo, %2, %0;\n\t}"
            : "+f"(acc[8 * wd + e])
            : "r"(t), "h"(xc));
      }
    }
    // words [WL, 8): register byte-permute lookups
#pragma unroll
    for (int wd = WL; wd < 8; ++wd) {
      uint32_t o[4];
      lookup8(cur[wd], L, H, o);
#pragma unroll
      for (int e = 0; e < 4; ++e) fma2_bf16(acc[8 * wd + 2 * e], acc[8 * wd + 2 * e + 1], o[e], xc);
    }
  }

  // ---- CTA reduction over the 8 warps (shared memory, swizzled float4 chunks)
  float4* my = red + ((size_t)wid * 32 + lane) * 16;
#pragma unroll
  for (int j4 = 0; j4 < 16; ++j4)
    my[j4 ^ (lane & 15)] = make_float4(acc[4 * j4], acc[4 * j4 + 1], acc[4 * j4 + 2], acc[4 * j4 + 3]);
  __syncthreads();
  const int t = threadIdx.x;
  const int src = t >> 3, j4a = (t & 7) * 2;  // columns [8t, 8t+8) of the strip
  float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
#pragma unroll
  for (int w = 0; w < WARPS; ++w) {
    const float4* row = red + ((size_t)w * 32 + src) * 16;
    const float4 a = row[j4a ^ (src & 15)], b = row[(j4a + 1) ^ (src & 15)];
    s0.x += a.x; s0.y += a.y; s0.z += a.z; s0.w += a.w;
    s1.x += b.x; s1.y += b.y; s1.z += b.z; s1.w += b.w;
  }
  const int64_t col = (int64_t)strip * STRIP + 8 * t;
  const bool col_live = col < N;  // N % 64 == 0: 8-column groups are all-in or all-out
  if (col_live) {
    float4* dst = reinterpret_cast<float4*>(part + (int64_t)z * N + col);
    dst[0] = s0;
    dst[1] = s1;
  }
  __threadfence();
  __syncthreads();
  if (t == 0) last_flag = (atomicAdd(counters + strip, 1u) == (unsigned)(zc - 1)) ? 1u : 0u;
  __syncthreads();
  if (!last_flag) return;
  __threadfence();

  // ---- last CTA of the strip: partials in split order + LoRA, bf16 out
  if (rank > 0) {
    for (int j = t; j < rank; j += TPB) {
      float a = 0.0f;
      for (int zz = 0; zz < zt; ++zz) a += __ldcg(tpart + (int64_t)zz * rank + j);
      tsh[j] = s * a;
    }
    __syncthreads();
  }
  if (!col_live) return;
  float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int zz = 0; zz < zc; ++zz) {
    const float4* p = reinterpret_cast<const float4*>(part + (int64_t)zz * N + col);
    const float4 a = __ldcg(p), b = __ldcg(p + 1);
    o[0] += a.x; o[1] += a.y; o[2] += a.z; o[3] += a.w;
    o[4] += b.x; o[5] += b.y; o[6] += b.z; o[7] += b.w;
  }
  if (rank > 0) {
    float l[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < rank; ++j) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(l2 + (int64_t)j * N + col));
      const uint32_t uu[4] = {u.x, u.y, u.z, u.w};
      const float tj = tsh[j];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        l[2 * e] = fmaf(tj, __uint_as_float(uu[e] << 16), l[2 * e]);
        l[2 * e + 1] = fmaf(tj, __uint_as_float(uu[e] & 0xFFFF0000u), l[2 * e + 1]);
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] += l[e];
  }
  uint4 out;
  out.x = pack_bf16x2(o[0], o[1]);
  out.y = pack_bf16x2(o[2], o[3]);
  out.z = pack_bf16x2(o[4], o[5]);
  out.w = pack_bf16x2(o[6], o[7]);
  *reinterpret_cast<uint4*>(y + col) = out;
}

// tpart[z][j] = sum over rows [128z, 128z+128) of x[k] l1[k][j]  (fp32)
__global__ void __launch_bounds__(TPB) lora_t_kernel(const __nv_bfloat16* __restrict__ x,
                                                     const __nv_bfloat16* __restrict__ l1, int64_t K, int rank,
                                                     float* __restrict__ tpart) {
  __shared__ float sh[8][512];
  const int z = blockIdx.x;
  const int pairs = rank / 2;
  const int pi = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int64_t k0 = (int64_t)z * 128;
  for (int p = pi; p < pairs; p += 32) {
    float a0 = 0.0f, a1 = 0.0f;
    for (int kk = rg; kk < 128; kk += 8) {
      const int64_t k = k0 + kk;
      if (k >= K) break;
      const float xv = __bfloat162float(x[k]);
      const uint32_t u = __ldg(reinterpret_cast<const uint32_t*>(l1 + k * rank) + p);
      a0 = fmaf(xv, __uint_as_float(u << 16), a0);
      a1 = fmaf(xv, __uint_as_float(u & 0xFFFF0000u), a1);
    }
    sh[rg][2 * p] = a0;
    sh[rg][2 * p + 1] = a1;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < rank; j += TPB) {
    float a = 0.0f;
#pragma unroll
    for (int g = 0; g < 8; ++g) a += sh[g][j];
    tpart[(int64_t)z * rank + j] = a;
  }
}

}  // namespace gemv
}  // namespace qlrt

using namespace qlrt;

extern "C" {

size_t qlrt_gemv_workspace_bytes(int64_t k_in, int64_t n_out, int rank) {
  return gemv::ws_bytes(k_in, n_out, rank);
}

qlrt_status qlrt_nf4_gemv(const qlrt_nf4_weight* w, const void* x, const void* xa, const void* l1, const void* l2,
                          int rank, float s, void* y, void* workspace, void* stream) {
  if (!w || !w->codes || !w->dq_codes || !w->c1 || !w->mu || w->k_in <= 0 || w->n_out <= 0 || (w->n_out % 64) ||
      !x || !y || !workspace || rank < 0 || rank > 512)
    return QLRT_ERR_ARG;
  if ((((uintptr_t)w->codes) & 31) || (((uintptr_t)y) & 15)) return QLRT_ERR_ARG;
  if (w->blocksize2 <= 0 || (w->blocksize2 & (w->blocksize2 - 1))) return QLRT_ERR_UNSUPPORTED;
  if (rank > 0 && (!l1 || !l2 || (rank % 8) || (((uintptr_t)l2) & 15) || (((uintptr_t)l1) & 3)))
    return QLRT_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t K = w->k_in, N = w->n_out;
  const gemv::Plan p = gemv::plan(K, N);
  uint8_t* ws = (uint8_t*)workspace;
  float* part = (float*)ws;
  float* tpart = (float*)(ws + gemv::align256((size_t)p.zc * N * 4));
  unsigned* counters = (unsigned*)(ws + gemv::align256((size_t)p.zc * N * 4) +
                                   gemv::align256((size_t)p.zt * (rank > 0 ? rank : 1) * 4));
  if (cudaMemsetAsync(counters, 0, (size_t)p.strips * 4, st) != cudaSuccess) return QLRT_ERR_CUDA;
  if (rank > 0)
    gemv::lora_t_kernel<<<p.zt, gemv::TPB, 0, st>>>((const __nv_bfloat16*)(xa ? xa : x), (const __nv_bfloat16*)l1, K, rank,
                                                    tpart);
  gemv::Vals32 v;
  for (int i = 0; i < 16; ++i) v.v[i] = (float)w->values[i];
  const int smem = gemv::WARPS * 32 * 16 * (int)sizeof(float4);  // 64 KB
  const int sh = __builtin_ctz((unsigned)w->blocksize2);
  const int wl = policy(P_GEMV_WL) < 0 ? 6 : policy(P_GEMV_WL);
#define QLRT_GEMV(WLV)                                                                                            \
  do {                                                                                                            \
    static bool attr = false;                                                                                     \
    if (!attr) {                                                                                                  \
      if (cudaFuncSetAttribute(gemv::gemv_nf4_kernel<WLV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != \
          cudaSuccess)                                                                                            \
        return QLRT_ERR_CUDA;                                                                                     \
      attr = true;                                                                                                \
    }                                                                                                             \
    gemv::gemv_nf4_kernel<WLV><<<dim3(p.strips, p.zc), gemv::TPB, smem, st>>>(                                    \
        w->codes, w->dq_codes, w->c1, w->mu, sh, w->spec, v, K, N, (const unsigned short*)x, part, counters,     \
        tpart, p.zt, (const __nv_bfloat16*)l2, rank, s, (__nv_bfloat16*)y);                                       \
  } while (0)
  switch (wl) {
    case 0: QLRT_GEMV(0); break;
    case 4: QLRT_GEMV(4); break;
    case 5: QLRT_GEMV(5); break;
    case 8: QLRT_GEMV(8); break;
    default: QLRT_GEMV(6); break;
  }
#undef QLRT_GEMV
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

}  // extern "C"
