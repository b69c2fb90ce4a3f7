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

#include <type_traits>

#include <cuda_fp16.h>

#include "qlrt_common.cuh"
#include "sm100_ptx.cuh"

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
#pragma unroll 8
      for (int zz = 0; zz < zt; ++zz) a += __ldcg(tpart + (int64_t)zz * rank + j);
      tsh[j] = s * a;
    }
    __syncthreads();
  }
  if (!col_live) return;
  float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
  for (int zz = 0; zz < zc; ++zz) {
    const float4* p = reinterpret_cast<const float4*>(part + (int64_t)zz * N + col);
    const float4 a = __ldcg(p), b = __ldcg(p + 1);
    o[0] += a.x; o[1] += a.y; o[2] += a.z; o[3] += a.w;
    o[4] += b.x; o[5] += b.y; o[6] += b.z; o[7] += b.w;
  }
  if (rank > 0) {
    float l[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
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

// ---------------------------------------------------------------------------
// Tensor-core GEMV (default): the decode is the bound of the kernel above
// (~5 SASS per weight for a bf16(v c) table rebuilt per block + byte-permute
// lookups + one FHFMA per weight).  Here the per-block constant moves to the
// other operand and the lookup becomes one PRMT + one LDS per TWO weights:
//
//   y_j = sum_k x_k W[k][j] = sum_k (x_k c_{k,b(j)}) v(code[k][j])
//
// * A operand (mma.sync m16n8k16, f16 in, f32 accumulate) = the codebook
//   values v of 16 columns x 16 rows, read from a fixed 256-entry table of
//   fp16 pairs {v(lo nibble), v(hi nibble)} indexed by a byte that holds the
//   codes of rows k and k+1 of one column (the fragment pairs along K).  The
//   table has a private column per lane (entry e at e*256 + lane*4: bank =
//   lane, no conflicts) at a 64 KB-aligned shared address, so the byte ->
//   address step is a single PRMT that drops the index byte into bits 8-15 of
//   the lane's column address.
// * B operand = a_k = x_k c_{k,b} * 2^-E as an fp16 hi/lo pair (B columns
//   2b / 2b+1 for the warp's two 64-column blocks b); the D rows of an m-tile
//   whose block matches the B column pair hold the result (the rest of the
//   16x8 tile is free compute).  c is the exact dq_decompress constant
//   (fp64, doublequant.py:190-195); E is one power of two per CTA (max|x|
//   over the CTA's rows times the largest constant its second-level blocks
//   allow) so that |a 2^-E| < 2^15 fits fp16; partials are scaled back
//   exactly.
// Precision: W enters as fp16(v) * c (v rounded to 11 bits, a to ~22 bits),
// i.e. closer to the reference's float32 W = f32(dequantize(q)) than the
// bf16 W of the tensor-core GEMM (GEMV tolerance).
//
// Data movement: a stage = 32 rows x 2048 columns (1 KB of codes per row)
// arrives as ONE 3-d TMA box [8 column groups][32 rows][128 B] (128B
// swizzle: conflict-free 8-byte reads; 2 KB boxes were TMA-issue bound at
// ~12 GB/s per SM), the stage's DQ bytes, x and c1 ride along as cp.async
// on the same mbarrier; a producer warp keeps NST = 3 stages (96 KB) in
// flight.  Units = (strip of 2048 columns, 32-row stage), split evenly over one CTA per SM in
// strip-major order (stream-K style: a CTA covers <= 2-3 strip segments).
// 16 warps: warp w owns columns [128 w, +128) of the strip (box w >> 1, half
// w & 1) and all 32 rows (two k16 halves) of each stage; lane (g, t) reads 8 bytes (16
// columns) of rows 2t, 2t+1, 2t+8, 2t+9.  A CTA flushes a strip segment as
// an fp32 partial; the last segment of a strip (atomic ticket) sums the
// partials in CTA order (deterministic), adds the LoRA term and writes bf16
// y.  The prep kernel (ticket reset, LoRA partials) is the PDL predecessor:
// the main grid waits for it only at its first flush.
namespace gemv2 {

#ifdef QLRT_GEMV_TL  // per-CTA globaltimer timeline (tools/gemv_tl.py); not in the product build
__device__ unsigned long long g_gemv_tl[kNumSMs][16];
__device__ unsigned long long g_gemv_tl_prep[2];  // [min start, max end] of the prep kernel
#define TLSET(slot, v) g_gemv_tl[blockIdx.x % kNumSMs][slot] = (unsigned long long)(v)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#else
#define TLSET(slot, v)
#endif
#ifndef QLRT_GEMV_EVICT_FIRST
#define QLRT_GEMV_EVICT_FIRST 1
#endif
constexpr int CWARPS = 16;  // consumer warps
constexpr int PWARP = CWARPS;  // + one producer warp (TMA + aux copies)
constexpr int TPB = (CWARPS + 1) * 32;
constexpr int CTHREADS = CWARPS * 32;
constexpr int STRIP = 2048;  // columns per strip = 8 TMA boxes of 128 B
constexpr int ROWS = 32;     // rows per stage (= unit): two k16 halves per stage
constexpr int NST = 3;  // stages in flight (32 KB each) = a_k input prefetch depth (static ring slots)
constexpr int STAGE = ROWS * STRIP / 2;  // 32 KB
// shared layout: the CTA's dynamic window starts a few KB into the 228 KB;
// the table sits at the 64 KB boundary, NFRONT stages + the scratch fill the
// gap in front of it, the other stages follow it
constexpr int NFRONT = 1;
constexpr int SMEM = 65536 + 65536 + (NST - NFRONT) * STAGE;

struct Geo {
  int64_t K, N, nbr, chunks, strips, units;
  int grid;
};

static Geo geo(int64_t K, int64_t N, int sms) {
  Geo g;
  g.K = K;
  g.N = N;
  g.nbr = N / 64;
  g.chunks = cdiv(K, ROWS);
  g.strips = cdiv(N, STRIP);
  g.units = g.chunks * g.strips;
  g.grid = (int)(g.units < sms ? g.units : sms);
  return g;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
// workspace: [partials (grid + strips) x STRIP f32][tpart zt x r f32][counters strips u32]
static size_t part_off() { return 0; }
static size_t tpart_off(const Geo& g) { return part_off() + align256((size_t)(g.grid + g.strips) * STRIP * 4); }
static size_t cnt_off(const Geo& g, int r) {
  return tpart_off(g) + align256((size_t)cdiv(g.K, 128) * (r > 0 ? r : 1) * 4);
}
static size_t ws_bytes(int64_t K, int64_t N, int r) {
  const Geo g = geo(K, N, kNumSMs);
  return cnt_off(g, r) + align256((size_t)g.strips * 4);
}

// first / last CTA covering strip s when CTA i owns units [i U / G, (i+1) U / G)
__device__ __forceinline__ int first_cta(int64_t s, int64_t C, int64_t U, int64_t G) {
  return (int)(((s * C + 1) * G + U - 1) / U) - 1;
}
__device__ __forceinline__ int last_cta(int64_t s, int64_t C, int64_t U, int64_t G) {
  return (int)(((s + 1) * C * G + U - 1) / U) - 1;
}

// prep (one launch, PDL predecessor of the main kernel, which waits for it
// only at its first strip flush): block 0 zeroes the strip tickets; blocks
// >= 1 compute the LoRA partials tpart[z][j] = sum_{k in [128 z, 128 z + 128)}
// xa_k l1[k][j] (8 columns per thread, 16-byte loads, all rows in flight)
__global__ void __launch_bounds__(256) prep_kernel(int64_t K, const __nv_bfloat16* __restrict__ xa,
                                                  const __nv_bfloat16* __restrict__ l1, int rank,
                                                  float* __restrict__ tpart, unsigned* __restrict__ counters,
                                                  int strips) {
  // launched programmatically behind whatever precedes it (its launch overlaps
  // that grid's tail): wait for it, and only then release the main grid, so
  // the main grid still starts after all prior work completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef QLRT_GEMV_TL
  if (threadIdx.x == 0) atomicMin(&g_gemv_tl_prep[0], gtimer());
  struct TlEnd {
    __device__ ~TlEnd() { if (threadIdx.x == 0) atomicMax(&g_gemv_tl_prep[1], gtimer()); }
  } tl_end;
#endif
  __shared__ float sh[256 * 8];
  const int tid = threadIdx.x;
  if (blockIdx.x == 0) {
    for (int i = tid; i < strips; i += 256) counters[i] = 0u;
    return;
  }
  const int z = blockIdx.x - 1;
  const int cpr = rank / 8;          // 16-byte column groups per row
  const int rpp = 256 / cpr;         // rows per pass
  const int cg = tid % cpr, rr = tid / cpr;
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (rr < rpp) {
    for (int k0 = z * 128 + rr; k0 < z * 128 + 128 && k0 < K; k0 += rpp) {
      const float xv = __bfloat162float(xa[k0]);
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(l1 + (int64_t)k0 * rank) + cg);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[2 * e] = fmaf(xv, __uint_as_float(w[e] << 16), a[2 * e]);
        a[2 * e + 1] = fmaf(xv, __uint_as_float(w[e] & 0xFFFF0000u), a[2 * e + 1]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) sh[tid * 8 + e] = a[e];
  __syncthreads();
  for (int j = tid; j < rank; j += 256) {
    float acc = 0.0f;
    for (int q = 0; q < rpp; ++q) acc += sh[(q * cpr + j / 8) * 8 + (j & 7)];
    tpart[(int64_t)z * rank + j] = acc;
  }
}

__device__ __forceinline__ uint32_t lds(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
// (a & 0x0F0F0F0F) | (b & 0xF0F0F0F0) as one LOP3
__device__ __forceinline__ uint32_t nib_merge(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "r"(0x0F0F0F0Fu));
  return d;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void cbar() {  // all 16 warps (named barrier 1)
  asm volatile("bar.sync 1, %0;" ::"n"(CTHREADS) : "memory");
}
// 4- / 16-byte async copies into the stage's aux slot; src_size 0 -> zero fill
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(ptx::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

struct Vals16 {
  float v[16];
};

// last segment of a strip: partials in CTA order + LoRA, bf16 out.  Every
// sum keeps a fixed order (deterministic); the loads of a sum are issued
// together (unrolled), not one dependent L2 round trip per term.
__device__ __noinline__ void finalize_strip(int64_t strip, int f, int l, int64_t N, const float* __restrict__ part,
                                            const float* __restrict__ tpart, int zt,
                                            const __nv_bfloat16* __restrict__ l2, int rank, float s,
                                            __nv_bfloat16* __restrict__ y, float* tsh) {
  __shared__ float tred[8][64];
  const int tid = threadIdx.x;
  __threadfence();
  if (rank > 0) {
    // T[j] = s * sum_z tpart[z][j]: 8 interleaved partial sums per j, combined in order
    const int jj = tid & 63, q = tid >> 6;
    for (int j0 = 0; j0 < rank; j0 += 64) {
      const int j = j0 + jj;
      float a = 0.0f;
      if (j < rank) {
        for (int z0 = q; z0 < zt; z0 += 64) {  // 8 loads in flight, summed in order
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = z0 + 8 * e < zt ? __ldcg(tpart + (int64_t)(z0 + 8 * e) * rank + j) : 0.f;
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (z0 + 8 * e < zt) a += v[e];
        }
      }
      tred[q][jj] = a;
      cbar();
      if (tid < 64 && j0 + tid < rank) {
        float t = 0.0f;
#pragma unroll
        for (int g = 0; g < 8; ++g) t += tred[g][tid];
        tsh[j0 + tid] = s * t;
      }
      cbar();
    }
  }
  // 4 consecutive columns per thread (STRIP = 4 * CTHREADS)
  const int c = 4 * tid;
  const int64_t col = strip * STRIP + c;
  if (col < N) {  // N % 64 == 0: 4-column groups are all-in or all-out
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    const float* pp = part + (int64_t)(f + strip) * STRIP + c;
    // 16 predicated loads in flight, then the adds in CTA order (a runtime
    // trip-count loop would run its remainder one L2 round trip at a time,
    // ~1-3 us each while other CTAs still stream)
    for (int i0 = f; i0 <= l; i0 += 16, pp += 16 * STRIP) {
      float4 v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        v[j] = i0 + j <= l ? __ldcg(reinterpret_cast<const float4*>(pp + j * STRIP)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (i0 + j <= l) {
          o[0] += v[j].x; o[1] += v[j].y; o[2] += v[j].z; o[3] += v[j].w;
        }
    }
    if (rank > 0) {
      float la[4] = {0.f, 0.f, 0.f, 0.f};
      const __nv_bfloat16* lp = l2 + col;
#pragma unroll 16
      for (int j = 0; j < rank; ++j, lp += N) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(lp));
        const float tj = tsh[j];
        la[0] = fmaf(tj, __uint_as_float(u.x << 16), la[0]);
        la[1] = fmaf(tj, __uint_as_float(u.x & 0xFFFF0000u), la[1]);
        la[2] = fmaf(tj, __uint_as_float(u.y << 16), la[2]);
        la[3] = fmaf(tj, __uint_as_float(u.y & 0xFFFF0000u), la[3]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) o[e] += la[e];
    }
    uint2 out;
    out.x = pack_bf16x2(o[0], o[1]);
    out.y = pack_bf16x2(o[2], o[3]);
    *reinterpret_cast<uint2*>(y + col) = out;
  }
  cbar();
}

// per-stage aux slot: DQ bytes [32 rows][32 blocks], x [32], c1 [32 rows][2]
constexpr int AUX_DQ = 0, AUX_X = 1024, AUX_C1 = 1088, AUX = 1408;

__global__ void __launch_bounds__(TPB, 1)
    gemv_mma_kernel(const __grid_constant__ CUtensorMap tm_codes, const uint8_t* __restrict__ dq_codes,
                    const float* __restrict__ c1, int64_t n2, const float* __restrict__ mu, int bs2_shift,
                    qlrt_fp8spec sp, Vals16 vals, float maxdec, int64_t K, int64_t N,
                    const unsigned short* __restrict__ x, float* __restrict__ part, unsigned* __restrict__ counters,
                    const float* __restrict__ tpart, int zt,
                    const __nv_bfloat16* __restrict__ l2, int rank, float s, __nv_bfloat16* __restrict__ y) {
  extern __shared__ __align__(1024) uint8_t dyn[];
  __shared__ float tsh[512];
  __shared__ unsigned last_flag;
  __shared__ float scales[2];
  __shared__ uint32_t v16[16];
  __shared__ unsigned red_max[CWARPS][2];
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t nbr = N / 64, chunks = cdiv(K, ROWS), strips = cdiv(N, STRIP), units = chunks * strips;
  const int G = (int)gridDim.x;
  const int64_t ub = (int64_t)blockIdx.x * units / G, ue = (int64_t)(blockIdx.x + 1) * units / G;
  const int nunits = (int)(ue - ub);
  // mu (a DRAM read that would otherwise queue behind the code stream): issued first
  float mu_f;
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(mu_f) : "l"(mu));
#ifdef QLRT_GEMV_TL
  unsigned long long tl_wait = 0;
  if (threadIdx.x == 0) { TLSET(0, gtimer()); TLSET(7, nunits); }
#endif

  // ---- shared layout: 64 KB table at the first 64 KB-aligned address;
  // 1 KB-aligned stages, the aux ring and the fp8 LUT around it
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(dyn);
  const uint32_t tab = (base + 65535u) & ~65535u;
  const uint32_t front = (base + 1023u) & ~1023u;
  const uint32_t back = tab + 65536u;
  const uint32_t aux0 = front + NFRONT * STAGE;
  const uint32_t lut_a = aux0 + NST * AUX;
  if (tab < lut_a + 2048u) __trap();  // (static smem grew: re-plan the layout)
  float* lut = reinterpret_cast<float*>(dyn + (lut_a - base));  // fp8 code -> value (exact in fp32)

  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      ptx::mbar_init(&full[i], 1 + 32);  // TMA tx arrive + warp 0's cp.async arrivals
      ptx::mbar_init(&empty[i], CWARPS);
    }
    ptx::fence_mbar_init();
  }
  if (tid < 16) v16[tid] = (uint32_t)__half_as_ushort(__float2half_rn(vals.v[tid]));
  if (tid < 256) lut[tid] = (float)fp8_decode_fast(tid, sp);
  __syncthreads();
#ifdef QLRT_GEMV_TL
  if (tid == 0) TLSET(10, gtimer());
#endif

  // ---- stage issue (warp 0; the codes and a_k inputs never depend on the
  // prep kernel): one TMA box of codes + the DQ bytes, x and c1 of the 32 rows
  int64_t ps = ub / chunks, pc = ub - ps * chunks;
#if QLRT_GEMV_EVICT_FIRST
  uint64_t evict_first;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(evict_first));
#endif
  auto slot_addr = [&](int sl) -> uint32_t {
    return sl < NFRONT ? front + (uint32_t)sl * STAGE : back + (uint32_t)(sl - NFRONT) * STAGE;
  };
  auto issue = [&](int sl) {  // called by all 32 lanes of warp 0
    const int64_t r0 = pc * ROWS;
    if (lane == 0) {  // one 3-d box [8 column groups][32 rows][128 B] (OOB groups zero-filled)
      ptx::mbar_arrive_expect_tx(&full[sl], (uint32_t)STAGE);
#if QLRT_GEMV_EVICT_FIRST
      // the codes are read once: evict-first in L2, so the stream does not
      // push out what is reused (x, c1, partials, this kernel's own code)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
          "%4, %5}], [%2], %6;" ::"r"(slot_addr(sl)),
          "l"(reinterpret_cast<uint64_t>(&tm_codes)), "r"(ptx::smem_u32(&full[sl])), "r"(0), "r"((int)r0),
          "r"((int)(ps * 8)), "l"(evict_first)
          : "memory");
#else
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
              slot_addr(sl)),
          "l"(reinterpret_cast<uint64_t>(&tm_codes)), "r"(ptx::smem_u32(&full[sl])), "r"(0), "r"((int)r0),
          "r"((int)(ps * 8))
          : "memory");
#endif
    }
    const uint32_t ax = aux0 + (uint32_t)sl * AUX;
    const int64_t jb0 = ps * 32;
#ifndef QLRT_GEMV_NOAUX
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // DQ bytes: 32 rows x 8 groups of 4 blocks
      const int p = lane + 32 * j, r = p >> 3, q = p & 7;
      const int64_t jb = jb0 + 4 * q;
      cp_async4(ax + AUX_DQ + r * 32 + q * 4, dq_codes + (r0 + r) * nbr + jb, jb < nbr);
    }
    if (lane < 4) cp_async16(ax + AUX_X + lane * 16, x + r0 + lane * 8, true);
#pragma unroll
    for (int which = 0; which < 2; ++which) {  // c1 of row lane: the (<= 2) second-level blocks its 32 blocks span
      const int64_t ic = (((r0 + lane) * nbr + jb0) >> bs2_shift) + which;
      cp_async4(ax + AUX_C1 + lane * 8 + which * 4, c1 + ic, ic < n2);
    }
#endif
    cp_async_arrive(&full[sl]);
    if (++pc == chunks) {
      pc = 0;
      ++ps;
    }
  };
  if (wid == PWARP) {
    if (lane == 0) ptx::prefetch_tmap(&tm_codes);
    for (int i = 0; i < nunits; ++i) {
      const int sl = i % NST;
      if (i >= NST) ptx::mbar_wait(&empty[sl], (uint32_t)((i / NST) - 1) & 1u);
      issue(sl);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#ifdef QLRT_GEMV_TL
    if (lane == 0) TLSET(6, gtimer());
#endif
    return;
  }

  // ---- this CTA's scale inputs (x, c1 of its rows; see below), loaded first
  // so their latency overlaps the table build
  const int64_t nrows_cta = (int64_t)nunits * ROWS;
  auto scale_item = [&](int64_t i, unsigned& xv, unsigned& c0, unsigned& c1v) {
    const int64_t uu = ub + i / ROWS, st = uu / chunks;
    const int64_t r = (uu - st * chunks) * ROWS + i % ROWS;
    const int64_t ic = (r * nbr + st * 32) >> bs2_shift;
    xv = (unsigned)__ldg(x + r) & 0x7FFFu;
    c0 = ic < n2 ? __float_as_uint(__ldg(c1 + ic)) & 0x7FFFFFFFu : 0u;
    c1v = ic + 1 < n2 ? __float_as_uint(__ldg(c1 + ic + 1)) & 0x7FFFFFFFu : 0u;
  };
  constexpr int SCALE_IT = 2;
  unsigned sx[SCALE_IT], s0[SCALE_IT], s1[SCALE_IT];
#pragma unroll
  for (int it = 0; it < SCALE_IT; ++it) {
    sx[it] = s0[it] = s1[it] = 0u;
    if (tid + (int64_t)it * CTHREADS < nrows_cta) scale_item(tid + (int64_t)it * CTHREADS, sx[it], s0[it], s1[it]);
  }

  // ---- table: entry e = {fp16 v(e & 15), fp16 v(e >> 4)} in every lane's column
  // (16-byte stores: 4 lanes' copies at a time)
  for (int q = tid; q < 256 * 8; q += CTHREADS) {
    const int e = q >> 3, l4 = q & 7;
    const uint32_t ev = v16[e & 15] | (v16[e >> 4] << 16);
    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(tab + (uint32_t)e * 256u + (uint32_t)l4 * 16u),
                 "r"(ev));
  }

#ifdef QLRT_GEMV_TL
  if (tid == 0) TLSET(8, gtimer());
#endif
  // ---- the fp16 scale 2^-E of this CTA: max |a| 2^-E < 2^15 over the a_k
  // of its own rows (a = x c, c <= maxdec max c1 + max(mu, 0)).  x and c1
  // are inputs (ready when the grid starts: the prep grid in front of it is
  // not programmatic); reading them here, before the code stream fills the
  // memory queues, is cheaper than a dependent read of values from the
  // prep grid once the stream runs (~3 us under full load).
  // Partials are unscaled per CTA, so E need not agree across CTAs.
  const double mu_d = (double)mu_f;
  {
    unsigned mx = 0u, mc = 0u;
#pragma unroll
    for (int it = 0; it < SCALE_IT; ++it) {
      mx = sx[it] > mx ? sx[it] : mx;
      mc = s0[it] > mc ? s0[it] : mc;
      mc = s1[it] > mc ? s1[it] : mc;
    }
    for (int64_t i = tid + (int64_t)SCALE_IT * CTHREADS; i < nrows_cta; i += CTHREADS) {
      unsigned xv, c0, c1v;
      scale_item(i, xv, c0, c1v);
      mx = xv > mx ? xv : mx;
      mc = c0 > mc ? c0 : mc;
      mc = c1v > mc ? c1v : mc;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned p = __shfl_xor_sync(0xffffffffu, mx, o), q = __shfl_xor_sync(0xffffffffu, mc, o);
      mx = p > mx ? p : mx;
      mc = q > mc ? q : mc;
    }
    if (lane == 0) {
      red_max[wid][0] = mx;
      red_max[wid][1] = mc;
    }
    cbar();
#ifdef QLRT_GEMV_TL
    if (tid == 0) TLSET(13, gtimer());
#endif
    if (tid == 0) {
      for (int w2 = 1; w2 < CWARPS; ++w2) {
        mx = red_max[w2][0] > mx ? red_max[w2][0] : mx;
        mc = red_max[w2][1] > mc ? red_max[w2][1] : mc;
      }
      const double m =
          (double)__uint_as_float(mx << 16) * ((double)maxdec * (double)__uint_as_float(mc) + fmax(mu_d, 0.0));
      int e = 0;
      if (m > 0.0 && m < 1e300) {
        e = ilogb(m) - 14;
        e = e < -120 ? -120 : (e > 120 ? 120 : e);
      }
      scales[0] = ldexpf(1.0f, -e);
      scales[1] = ldexpf(1.0f, e);
    }
  }
  cbar();  // (also: the table is complete)
  const float sc = scales[0], unsc = scales[1];
#ifdef QLRT_GEMV_TL
  if (tid == 0) TLSET(1, gtimer());
#endif

  // ---- consumers: warp w owns columns [128 w, +128) of the strip (box w >> 1, half w & 1)
  const int g = lane >> 2, t = lane & 3;
  const int bx = wid >> 1, u = wid & 1;
  const uint32_t lanereg = tab + (uint32_t)lane * 4u;
  // this lane's 8 code bytes of rows 2t, 2t+1, 2t+8, 2t+9 inside box bx (128B swizzle)
  const int cidx = u * 4 + (g >> 1);
  // (half q of the stage = rows 16 q .. 16 q + 15: the same offsets + q * 2 KB,
  // since (r + 16) & 7 = r & 7 keeps the swizzle)
  uint32_t roff[4];
  {
    const int rr[4] = {2 * t, 2 * t + 1, 2 * t + 8, 2 * t + 9};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      roff[i] = (uint32_t)bx * (ROWS * 128) + (uint32_t)rr[i] * 128u + (uint32_t)((cidx ^ (rr[i] & 7)) << 4) +
                (uint32_t)(g & 1) * 8u;
  }
  // a_k of (rows a_r = lane & 15 and a_r + 16, block jl = 4 bx + 2 u + (lane >> 4) of the strip)
  const int a_r = lane & 15, jl = bx * 4 + u * 2 + (lane >> 4);
  const uint32_t a_dq = AUX_DQ + a_r * 32 + jl, a_x = AUX_X + a_r * 2, a_c = AUX_C1 + a_r * 8;
  int64_t cs = ub / chunks;
  // first-level block of the lane's row at the strip's first column: only its
  // offset inside a second-level block matters (which of the <= 2 c1 values
  // the lane's block uses), kept as a 32-bit residue
  const uint32_t bmask2 = (1u << bs2_shift) - 1u;
  uint32_t lo2 = (uint32_t)(((((ub - cs * chunks) * ROWS) + a_r) * nbr + cs * 32) & bmask2);
  bool jok = cs * 32 + jl < nbr;
  const uint32_t step2 = (uint32_t)((ROWS * nbr) & bmask2);
  const uint32_t half2 = (uint32_t)((16 * nbr) & bmask2);  // residue step to row a_r + 16

  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0f;

  int left = (int)((cs + 1) * chunks - ub);  // units of strip cs still to do
  const int src0 = ((g >> 1) & 1) * 16 + 2 * t;
  const uint32_t bsel = (g & 1) ? 0x7632u : 0x5410u;
  const uint32_t bmask = g < 4 ? 0xFFFFFFFFu : 0u;  // lanes g < 4 hold B column g
  int sl = 0;
  uint32_t par = 0u;
  bool waited_prep = false;  // prep (tickets, LoRA partials): waited for at the first flush
  for (int i = 0; i < nunits; ++i) {
    if (left == 0) {
      // ---- strip segment done: partial, ticket, maybe finalize
      if (!waited_prep) {  // prep: zeroed tickets, LoRA partials
        asm volatile("griddepcontrol.wait;" ::: "memory");
        waited_prep = true;
      }
      if (t == (g >> 2)) {  // useful D lanes: lane g holds columns 16 g + 2 mt (+1) of the warp's 128
        float* dst = part + (blockIdx.x + cs) * STRIP + wid * 128 + 16 * g;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
          *reinterpret_cast<float2*>(dst + 2 * mt) =
              make_float2((acc[mt][0] + acc[mt][1]) * unsc, (acc[mt][2] + acc[mt][3]) * unsc);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.0f;
      __threadfence();
      cbar();
      const int f = first_cta(cs, chunks, units, G), l = last_cta(cs, chunks, units, G);
      if (tid == 0) last_flag = (atomicAdd(counters + cs, 1u) == (unsigned)(l - f)) ? 1u : 0u;
      cbar();
      if (last_flag) finalize_strip(cs, f, l, N, part, tpart, zt, l2, rank, s, y, tsh);
      ++cs;
      left = (int)chunks;
      lo2 = (uint32_t)(((int64_t)a_r * nbr + cs * 32) & bmask2);
      jok = cs * 32 + jl < nbr;
    }
    --left;
#ifdef QLRT_GEMV_TL
    {
      const unsigned long long t0 = gtimer();
      ptx::mbar_wait(&full[sl], par);
      if (tid == 0) {
        const unsigned long long t1 = gtimer();
        tl_wait += t1 - t0;
        if (i == 0) TLSET(2, t1);
      }
    }
#else
    ptx::mbar_wait(&full[sl], par);
#endif
#ifdef QLRT_GEMV_DIAG  // data movement only (measurement build)
    if (lane == 0) ptx::mbar_arrive(&empty[sl]);
    if (++sl == NST) {
      sl = 0;
      par ^= 1u;
    }
    continue;
#endif
    const uint32_t sa = sl < NFRONT ? front + (uint32_t)sl * STAGE : back + (uint32_t)(sl - NFRONT) * STAGE;
    const uint32_t ax = aux0 + (uint32_t)sl * AUX;
    uint2 w[2][4];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int i2 = 0; i2 < 4; ++i2) w[q][i2] = lds64(sa + q * 2048u + roff[i2]);
    // a_k = x_k c_k 2^-E as an fp16 hi | lo pair, rows a_r (q = 0) and a_r + 16 (q = 1)
    uint32_t hv[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      uint32_t dqb, xb, c1b;
      asm volatile("ld.shared.u8 %0, [%1];" : "=r"(dqb) : "r"(ax + a_dq + q * 512u));
      asm volatile("ld.shared.u16 %0, [%1];" : "=r"(xb) : "r"(ax + a_x + q * 32u));
      const uint32_t which = (((lo2 + (q ? half2 : 0u)) & bmask2) + (uint32_t)jl) >> bs2_shift;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(c1b) : "r"(ax + a_c + q * 128u + which * 4u));
      // c = max(v_dq c1 + mu, 0) in one fp32 rounding (fma; the reference
      // rounds the fp64 value to fp32 -- equal except for a double-rounding
      // tie, far inside the GEMV tolerance)
      const float c = fmaxf(fmaf(lut[dqb], __uint_as_float(c1b), mu_f), 0.0f);
      const float a = jok ? (__uint_as_float(xb << 16) * c) * sc : 0.0f;
      const __half h = __float2half_rn(a);
      const float dl = a - __half2float(h);
      asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hv[q]) : "f"(dl), "f"(a));  // {lo = h, hi = f16(a - h)}
    }
    lo2 = (lo2 + step2) & bmask2;
    // index bytes: codes of rows (2t, 2t+1) resp. (2t+8, 2t+9) of one column
    uint32_t ie[2][2], io[2][2], je[2][2], jo[2][2];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t x0 = h ? w[q][0].y : w[q][0].x, x1 = h ? w[q][1].y : w[q][1].x;
        const uint32_t x2 = h ? w[q][2].y : w[q][2].x, x3 = h ? w[q][3].y : w[q][3].x;
        ie[q][h] = nib_merge(x0, x1 << 4);
        io[q][h] = nib_merge(x0 >> 4, x1);
        je[q][h] = nib_merge(x2, x3 << 4);
        jo[q][h] = nib_merge(x2 >> 4, x3);
      }
    // B fragments: lanes g < 4 take column n = g (block g >> 1, hi / lo by g & 1)
    uint32_t b0[2], b1[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t v0 = __shfl_sync(0xffffffffu, hv[q], src0);
      const uint32_t v1 = __shfl_sync(0xffffffffu, hv[q], src0 + 1);
      const uint32_t v2 = __shfl_sync(0xffffffffu, hv[q], src0 + 8);
      const uint32_t v3 = __shfl_sync(0xffffffffu, hv[q], src0 + 9);
      b0[q] = __byte_perm(v0, v1, bsel) & bmask;
      b1[q] = __byte_perm(v2, v3, bsel) & bmask;
    }
    // (the shuffles used every lane's aux bytes, the index bytes its codes:
    // release the slot)
    if (lane == 0) ptx::mbar_arrive(&empty[sl]);
    if (++sl == NST) {
      sl = 0;
      par ^= 1u;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint32_t sel = 0x7604u | ((uint32_t)b << 4);
          const uint32_t a0 = lds(__byte_perm(ie[q][h], lanereg, sel));
          const uint32_t a1 = lds(__byte_perm(io[q][h], lanereg, sel));
          const uint32_t a2 = lds(__byte_perm(je[q][h], lanereg, sel));
          const uint32_t a3 = lds(__byte_perm(jo[q][h], lanereg, sel));
          mma16816(acc[4 * h + b], a0, a1, a2, a3, b0[q], b1[q]);
        }
      }
  }
  // ---- last segment
#ifdef QLRT_GEMV_TL
  if (tid == 0) { TLSET(3, gtimer()); TLSET(5, tl_wait); }
#endif
  if (!waited_prep) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (t == (g >> 2)) {
    float* dst = part + (blockIdx.x + cs) * STRIP + wid * 128 + 16 * g;
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
      *reinterpret_cast<float2*>(dst + 2 * mt) =
          make_float2((acc[mt][0] + acc[mt][1]) * unsc, (acc[mt][2] + acc[mt][3]) * unsc);
  }
  __threadfence();
  cbar();
  const int f = first_cta(cs, chunks, units, G), l = last_cta(cs, chunks, units, G);
  if (tid == 0) last_flag = (atomicAdd(counters + cs, 1u) == (unsigned)(l - f)) ? 1u : 0u;
  cbar();
#ifdef QLRT_GEMV_TL
  if (tid == 0) { TLSET(11, gtimer()); TLSET(12, last_flag); }
#endif
  if (last_flag) finalize_strip(cs, f, l, N, part, tpart, zt, l2, rank, s, y, tsh);
#ifdef QLRT_GEMV_TL
  if (tid == 0) TLSET(4, gtimer());
#endif
}

// packed codes [K rows][N/2 bytes] as a 3-d uint8 tensor, box [8][32 rows][128 B], 128B swizzle
static bool make_tmap_codes(CUtensorMap* m, const void* base, int64_t row_bytes, int64_t rows) {
  typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  if (!fn || (((uintptr_t)base) & 15) || (row_bytes & 127)) return false;
  // 3-d view {128 B, rows, 128-B column groups}: one box = a whole stage
  cuuint64_t dims[3] = {128, (cuuint64_t)rows, (cuuint64_t)(row_bytes / 128)};
  cuuint64_t strides[2] = {(cuuint64_t)row_bytes, 128};
  cuuint32_t box[3] = {128, ROWS, 8};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace gemv2
}  // namespace qlrt

using namespace qlrt;

extern "C" {
#ifdef QLRT_GEMV_TL
// host: [kNumSMs][16] per-CTA slots, then the prep kernel's [start, end]; resets the prep pair
int qlrt_gemv_tl_fetch(unsigned long long* host) {
  if (cudaMemcpyFromSymbol(host, gemv2::g_gemv_tl, sizeof(gemv2::g_gemv_tl)) != cudaSuccess) return 1;
  if (cudaMemcpyFromSymbol(host + kNumSMs * 16, gemv2::g_gemv_tl_prep, 16) != cudaSuccess) return 1;
  const unsigned long long init[2] = {~0ull, 0ull};
  return cudaMemcpyToSymbol(gemv2::g_gemv_tl_prep, init, 16) == cudaSuccess ? 0 : 1;
}
#endif

size_t qlrt_gemv_workspace_bytes(int64_t k_in, int64_t n_out, int rank) {
  const size_t a = gemv::ws_bytes(k_in, n_out, rank), b = gemv2::ws_bytes(k_in, n_out, rank);
  return a > b ? a : b;
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
  CUtensorMap tmc;
  if (policy(P_GEMV_MMA) && (N % 256) == 0 && (K % gemv2::ROWS) == 0 && w->blocksize2 >= 32 &&
      (((uintptr_t)x) & 15) == 0 && gemv2::make_tmap_codes(&tmc, w->codes, N / 2, K)) {
    // tensor-core GEMV: prep (tickets, LoRA partials) then the
    // main kernel as its PDL dependent (prologue + first TMA loads overlap prep)
    int dev = 0, sms = kNumSMs;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // small weights: fewer CTAs with >= QLRT_GEMV_MIN_UNITS stages each (fewer
    // strip partials to sum; the per-CTA prologue amortized over more stages)
    const int64_t units_all = cdiv(K, gemv2::ROWS) * cdiv(N, gemv2::STRIP);
    const int mu_ = policy(P_GEMV_MIN_UNITS) > 0 ? policy(P_GEMV_MIN_UNITS) : 1;
    const int64_t want = cdiv(units_all, mu_);
    const gemv2::Geo g = gemv2::geo(K, N, (int)(want < sms ? want : sms));
    uint8_t* ws = (uint8_t*)workspace;
    float* part = (float*)(ws + gemv2::part_off());
    float* tpart = (float*)(ws + gemv2::tpart_off(g));
    unsigned* counters = (unsigned*)(ws + gemv2::cnt_off(g, rank));
    const int zt = (int)cdiv(K, 128);
    const double maxdec = fp8_max_value(w->spec.exp_bits, w->spec.mant_bits, w->spec.bias);
    const int64_t n2 = cdiv(K * (N / 64), (int64_t)w->blocksize2);
    {
      cudaLaunchConfig_t pc{};
      pc.gridDim = dim3((unsigned)(1 + (rank > 0 ? zt : 0)));
      pc.blockDim = dim3(256);
      pc.stream = st;
      cudaLaunchAttribute pa[1];
      pa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      pa[0].val.programmaticStreamSerializationAllowed = 1;
      pc.attrs = pa;
      pc.numAttrs = policy(P_PDL) ? 1 : 0;
      if (cudaLaunchKernelEx(&pc, gemv2::prep_kernel, K, (const __nv_bfloat16*)(xa ? xa : x),
                             (const __nv_bfloat16*)l1, rank, tpart, counters, (int)g.strips) != cudaSuccess)
        return QLRT_ERR_CUDA;
    }
    static std::atomic<unsigned long long> attr_mask{0};
    if (!(attr_mask.load() & (1ull << (dev & 63)))) {
      if (cudaFuncSetAttribute(gemv2::gemv_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gemv2::SMEM) !=
          cudaSuccess)
        return QLRT_ERR_CUDA;
      // both kernels at the full shared-memory carveout: no L1/smem
      // reconfiguration between the prep grid and the main grid
      cudaFuncSetAttribute(gemv2::gemv_mma_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaFuncSetAttribute(gemv2::prep_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      attr_mask.fetch_or(1ull << (dev & 63));
    }
    gemv2::Vals16 v;
    for (int i = 0; i < 16; ++i) v.v[i] = (float)w->values[i];
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)g.grid);
    cfg.blockDim = dim3(gemv2::TPB);
    cfg.dynamicSmemBytes = gemv2::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = policy(P_PDL) ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, gemv2::gemv_mma_kernel, tmc, w->dq_codes, w->c1, n2, w->mu,
                           (int)__builtin_ctz((unsigned)w->blocksize2), w->spec, v, (float)maxdec, K, N,
                           (const unsigned short*)x, part, counters, (const float*)tpart, zt,
                           (const __nv_bfloat16*)l2, rank, s, (__nv_bfloat16*)y) != cudaSuccess)
      return QLRT_ERR_CUDA;
    QLRT_CHECK_LAUNCH();
    return QLRT_OK;
  }
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
