// NF4 (any 4-bit codebook) block-wise quantize, double quantization and
// double-dequantize for sm_100a.  Restates, bit-exactly, the reference's
//   blockquant.quantize / dequantize / pack_codes / unpack_codes
//   (pkg/src/qlrt/blockquant.py:81-213) and
//   doublequant.dq_compress / dq_decompress (pkg/src/qlrt/doublequant.py:148-195).
// All kernels are HBM-bound streaming kernels: 128-bit coalesced loads and
// stores, grids sized in multiples of the 148 SMs.
#include <cstdlib>
#include <type_traits>

#include "qlrt_common.cuh"

namespace qlrt {

// ---------------------------------------------------------------------------
// code search: #{mids <= q} for q >= 0 (incl. -0.0), #{mids < q} for q < 0
// (blockquant.py:123-129).  Fast path in fp32 against brackets [lo_i, hi_i]
// that contain each midpoint with a wide margin; inside a bracket the code is
// re-decided from the fp64 quotient x / f64(c), exactly as the reference.
// ---------------------------------------------------------------------------
struct CodeTables {
  float lo[16];   // lo[n_mids..15] = +inf
  float hi[16];
  double mids[15];
  int n_mids;
};

__device__ __forceinline__ unsigned exact_code(double x, float c, const CodeTables& t) {
  double q = __ddiv_rn(x, (double)c);
  unsigned k = 0;
  if (q >= 0.0) {
    for (int i = 0; i < t.n_mids; ++i) k += (t.mids[i] <= q) ? 1u : 0u;
  } else {
    for (int i = 0; i < t.n_mids; ++i) k += (t.mids[i] < q) ? 1u : 0u;
  }
  return k;
}

__device__ __forceinline__ unsigned fast_code(double xd, float r, float c, const CodeTables& t) {
  // for fp64 inputs the fp32 rounding of x (2^-24 rel.) is far inside the bracket margin
  float q = __double2float_rn(xd) * r;
  unsigned j = (q > t.lo[7]) ? 8u : 0u;
  j += (q > t.lo[j + 3]) ? 4u : 0u;
  j += (q > t.lo[j + 1]) ? 2u : 0u;
  j += (q > t.lo[j]) ? 1u : 0u;
  // q in (lo[j-1], lo[j]]: certain unless it sits inside bracket j-1
  if (j > 0 && q < t.hi[j - 1]) return exact_code(xd, c, t);
  return j;
}

template <typename T> struct AccT { using type = float; };
template <> struct AccT<double> { using type = double; };

template <typename T>
__device__ __forceinline__ void load8(const T* __restrict__ x, int64_t i, int64_t n, typename AccT<T>::type v[8]);

template <>
__device__ __forceinline__ void load8<float>(const float* __restrict__ x, int64_t i, int64_t n, float v[8]) {
  if (i + 8 <= n) {
    float4 a = __ldg(reinterpret_cast<const float4*>(x + i));
    float4 b = __ldg(reinterpret_cast<const float4*>(x + i + 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (i + j < n) ? x[i + j] : 0.0f;
  }
}

template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* __restrict__ x, int64_t i, int64_t n,
                                                     float v[8]) {
  if (i + 8 <= n) {
    uint4 a = __ldg(reinterpret_cast<const uint4*>(x + i));
    uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[2 * j] = __uint_as_float(w[j] << 16);
      v[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (i + j < n) ? __bfloat162float(x[i + j]) : 0.0f;
  }
}

template <>
__device__ __forceinline__ void load8<double>(const double* __restrict__ x, int64_t i, int64_t n, double v[8]) {
  if (i + 8 <= n) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double2 a = __ldg(reinterpret_cast<const double2*>(x + i) + j);
      v[2 * j] = a.x;
      v[2 * j + 1] = a.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (i + j < n) ? x[i + j] : 0.0;
  }
}

__device__ __forceinline__ bool finite_v(float a) { return fabsf(a) <= 3.402823466e38f; }
__device__ __forceinline__ bool finite_v(double a) { return fabs(a) <= 1.7976931348623157e308; }
__device__ __forceinline__ float to_f32_const(float m) { return m; }
__device__ __forceinline__ float to_f32_const(double m) { return __double2float_rn(m); }

// Bin table for the code search.  q in [-1, 1] is cut into NBIN equal bins;
// every bin overlaps at most one midpoint bracket (the host checks the
// spacing), so  j = base[bin] + (q > lo[base])  and the result is certain
// iff  lower[j] <= q <= upper[j]  with lower[j] = hi[j-1], upper[j] = lo[j];
// otherwise (inside a bracket, or a bin-edge rounding case) the code is
// re-decided exactly in fp64.
#ifndef QLRT_NBIN
#define QLRT_NBIN 128  // small table: fewer shared-memory bank conflicts (1024: -5% quantize)
#endif
constexpr int NBIN = QLRT_NBIN;
struct BinTables {
  float2 bin[NBIN];      // (base code as float bits, lo[base])
  float2 bound[16];      // (hi[j-1] or -inf, lo[j] or +inf)
  double mids[15];
  int n_mids;
};

__device__ void build_bin_tables(BinTables& T, const qlrt_codebook4& cb) {
  const int n = cb.n_mids;
  for (int b = threadIdx.x; b < NBIN; b += blockDim.x) {
    const float qb = -1.0f + 2.0f * (float)b / (float)NBIN;  // bin start (exact)
    int base = 0;  // #{hi[i] <= qb}: hi ascending, unrolled (constant-bank operands)
#pragma unroll
    for (int i = 0; i < 15; ++i) base += (i < n && cb.hi[i] <= qb) ? 1 : 0;
    T.bin[b] = make_float2(__int_as_float(base), base < n ? cb.lo[base] : __int_as_float(0x7f800000));
  }
  if (threadIdx.x < 16) {
    const int j = threadIdx.x;
    T.bound[j] = make_float2(j == 0 ? __int_as_float(0xff800000) : (j <= n ? cb.hi[j - 1] : __int_as_float(0x7f800000)),
                             j < n ? cb.lo[j] : __int_as_float(0x7f800000));
    if (j < 15) T.mids[j] = cb.mids[j];
  }
  if (threadIdx.x == 0) T.n_mids = n;
}

__device__ __forceinline__ unsigned exact_code_t(double x, float c, const BinTables& t) {
  double q = __ddiv_rn(x, (double)c);
  unsigned k = 0;
  if (q >= 0.0) {
    for (int i = 0; i < t.n_mids; ++i) k += (t.mids[i] <= q) ? 1u : 0u;
  } else {
    for (int i = 0; i < t.n_mids; ++i) k += (t.mids[i] < q) ? 1u : 0u;
  }
  return k;
}

template <typename V>
__device__ __forceinline__ unsigned bin_code(V x, float r, float c, const BinTables& t) {
  const float q = (float)x * r;
  int b = __float2int_rd(fmaf(q, 0.5f * NBIN, 0.5f * NBIN));
  b = min(max(b, 0), NBIN - 1);
  const float2 e = t.bin[b];
  const unsigned j = (unsigned)__float_as_int(e.x) + (q > e.y ? 1u : 0u);
  const float2 bd = t.bound[j];
  if (!(q >= bd.x && q <= bd.y)) return exact_code_t((double)x, c, t);
  return j;
}

// fast-path code of one element; clears ok when q lies inside a midpoint
// bracket or on a bin-edge rounding case (the caller then redoes the group)
template <typename V>
__device__ __forceinline__ unsigned bin_j(V x, float r, const BinTables& t, bool& ok) {
  const float q = (float)x * r;
  int b = __float2int_rd(fmaf(q, 0.5f * NBIN, 0.5f * NBIN));
  b = min(max(b, 0), NBIN - 1);
  const float2 e = t.bin[b];
  const unsigned j = (unsigned)__float_as_int(e.x) + (q > e.y ? 1u : 0u);
  const float2 bd = t.bound[j];
  ok = ok && (q >= bd.x) && (q <= bd.y);
  return j;
}

template <typename T>
__device__ __forceinline__ void load8_stream(const T* __restrict__ x, int64_t i, float (&v)[8]);
template <>
__device__ __forceinline__ void load8_stream<float>(const float* __restrict__ x, int64_t i, float (&v)[8]) {
  uint32_t u[8];
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
               : "l"(x + i));
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(u[j]);
}
template <>
__device__ __forceinline__ void load8_stream<__nv_bfloat16>(const __nv_bfloat16* __restrict__ x, int64_t i,
                                                            float (&v)[8]) {
  uint4 a;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w)
               : "l"(x + i));
  const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v[2 * j] = __uint_as_float(w[j] << 16);
    v[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
  }
}

// Single-lookup bin table with a private column per lane (entry b of lane l
// at b * 256 + l * 8: bank = lane, conflict-free): float2 (lo', hi) where the
// low 4 mantissa bits of lo' carry the base code of the bin and lo' is the
// bracket's lower end moved outwards by <= 31 ulp (never inwards).  For q in
// the bin:  j = base + (q > lo'),  certain unless lo' < q < hi (then the
// group is re-decided exactly).  Bins a bracket does not touch hold lo' = 4.0
// (q > lo' never); bins that touch two or more brackets hold lo' = -4.0,
// hi = 4.0 (always re-decided).  Bin edges are widened by 2^-20 so the fp32
// bin index may be off by one at an edge.
constexpr int PBIN = 128;
constexpr float PS = 63.875f;  // |q| <= 1 + 2^-20 maps into [0.1, 127.9]: no clamp
__device__ void build_private_bins(uint32_t tab, const qlrt_codebook4& cb, uint2* ent) {
  // one entry per bin (PBIN threads), then replicated into every lane's column
  const int n = cb.n_mids;
  const float dlt = 9.5367431640625e-07f;  // 2^-20
  for (int b = threadIdx.x; b < PBIN; b += blockDim.x) {
    // bin b = floor(q * PS + 64) holds q in [(b - 64) / PS, (b - 63) / PS)
    const float qa = (float)(b - 64) / PS - dlt;
    const float qb = (float)(b - 63) / PS + dlt;
    int base = 0, hits = 0, hit = 0;
    for (int i = 0; i < n; ++i) {
      if (cb.hi[i] < qa) ++base;
      if (cb.lo[i] <= qb && cb.hi[i] >= qa) {
        ++hits;
        hit = i;
      }
    }
    uint32_t lo_b;
    float hi;
    if (hits == 0) {
      lo_b = __float_as_uint(4.0f) | (uint32_t)base;
      hi = 4.0f;
    } else if (hits == 1) {
      const uint32_t bits = __float_as_uint(cb.lo[hit]);
      lo_b = ((bits >> 31) ? ((bits + 16u) & ~15u) : ((bits - 16u) & ~15u)) | (uint32_t)base;
      hi = cb.hi[hit];
    } else {
      lo_b = __float_as_uint(-4.0f) | (uint32_t)base;
      hi = 4.0f;
    }
    ent[b] = make_uint2(lo_b, __float_as_uint(hi));
  }
  __syncthreads();
  for (int q = threadIdx.x; q < PBIN * 32; q += blockDim.x) {
    const int b = q >> 5, l = q & 31;
    const uint2 e = ent[b];
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(tab + (uint32_t)b * 256u + (uint32_t)l * 8u), "r"(e.x),
                 "r"(e.y));
  }
}

// code of element k of the group added into word (fields do not overlap:
// word += code << 4k is one IMAD); bad |= (q inside the bin's bracket)
template <int K>
__device__ __forceinline__ void pbin_acc(float x, float r, uint32_t lanecol, uint32_t& word, bool& bad) {
  const float q = x * r;
  const uint32_t b = (uint32_t)__float2int_rd(fmaf(q, PS, 64.0f));
  uint32_t lo_b, hi_b;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lo_b), "=r"(hi_b) : "r"(lanecol + (b << 8)));
  const bool above = q > __uint_as_float(lo_b);
  bad = bad || (above && q < __uint_as_float(hi_b));
  word += ((lo_b & 15u) + (above ? 1u : 0u)) * (1u << (4 * K));
}

// Phase A, fp32 / bf16 input, blocksize 64, n % 64 == 0 (whole blocks): the
// streaming version.  8 lanes per block as below, a persistent grid, the next
// two groups' 32 B (fp32: one 256-bit load each) in flight while the current one is
// coded, and a branch-free fast path per element with one group-wide check
// (bracket hits are re-decided exactly, rarely).
template <typename T>
#ifndef QLRT_Q_MINB
#define QLRT_Q_MINB 4  // 4 resident CTAs per SM (62 registers, no spills since the alternating group buffers): +3% over 3
#endif
__global__ void __launch_bounds__(256, QLRT_Q_MINB) quantize64_stream_kernel(const T* __restrict__ x, int64_t n_groups,
                                                                qlrt_codebook4 cb, uint32_t* __restrict__ codes,
                                                                float* __restrict__ absmax,
                                                                unsigned long long* __restrict__ first_bad) {
  __shared__ BinTables t;
  __shared__ uint2 pent[PBIN];
  extern __shared__ __align__(16) uint8_t ptab[];  // PBIN x 32 lanes x 8 B
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // two group buffers in flight, used alternately (no register rotation);
  // a lane past the end keeps stale (finite or ignored) values: it reports
  // nothing and stores nothing, and its 8-lane group only shuffles with itself
  float va[8], vb[8];
  if (g < n_groups) load8_stream<T>(x, g * 8, va);
  if (g + stride < n_groups) load8_stream<T>(x, (g + stride) * 8, vb);
  build_bin_tables(t, cb);
  const uint32_t tab = (uint32_t)__cvta_generic_to_shared(ptab);
  build_private_bins(tab, cb, pent);
  const uint32_t lanecol = tab + (uint32_t)lane * 8u;
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // (the DQ chunk sums wait for our completion)
  const unsigned pad = (unsigned)cb.pad_code;
  auto body = [&](const float (&v)[8], int64_t gg) {
    const bool act = gg < n_groups;
    unsigned mb = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) mb = max(mb, __float_as_uint(v[j]) & 0x7FFFFFFFu);
    if (act && mb >= 0x7F800000u) {  // inf / NaN: first bad flat index
      unsigned long long bad = ~0ull;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if ((__float_as_uint(v[j]) & 0x7FFFFFFFu) >= 0x7F800000u) bad = min(bad, (unsigned long long)(gg * 8 + j));
      atomicMin(first_bad, bad);
    }
    mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, 1));
    mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, 2));
    mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, 4));
    if (!act) return;
    const float c = __uint_as_float(mb);
    uint32_t word;
    if (c > 0.0f) {
      const float r = __frcp_rn(c);
      bool bad = !(r <= 3.402823466e38f);  // subnormal c: 1/c overflows -> exact path
      word = 0;
      pbin_acc<0>(v[0], r, lanecol, word, bad);
      pbin_acc<1>(v[1], r, lanecol, word, bad);
      pbin_acc<2>(v[2], r, lanecol, word, bad);
      pbin_acc<3>(v[3], r, lanecol, word, bad);
      pbin_acc<4>(v[4], r, lanecol, word, bad);
      pbin_acc<5>(v[5], r, lanecol, word, bad);
      pbin_acc<6>(v[6], r, lanecol, word, bad);
      pbin_acc<7>(v[7], r, lanecol, word, bad);
      if (bad) {
        const bool fast_ok = r <= 3.402823466e38f;
        word = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          word |= (fast_ok ? bin_code(v[j], r, c, t) : exact_code_t((double)v[j], c, t)) << (4 * j);
      }
    } else {
      word = pad * 0x11111111u;
    }
    codes[gg] = word;
    if ((threadIdx.x & 7) == 0) absmax[gg >> 3] = c;
  };
  // n_groups % 8 == 0 and stride % 8 == 0: 8-lane groups are all-in or all-out,
  // and the trip count is warp-uniform (the shuffles need every lane)
  for (int64_t gb = g - lane; gb < n_groups; gb += 2 * stride, g += 2 * stride) {
    body(va, g);
    if (g + 2 * stride < n_groups) load8_stream<T>(x, (g + 2 * stride) * 8, va);
    if (gb + stride >= n_groups) break;
    body(vb, g + stride);
    if (g + 3 * stride < n_groups) load8_stream<T>(x, (g + 3 * stride) * 8, vb);
  }
}

// Phase A, blocksize 64: 8 consecutive lanes own one 64-block, 8 elements
// each (two 16B loads for fp32, one for bf16, four for fp64); absmax by 3
// xor-shuffles; 8 codes -> one 32-bit packed store.
template <typename T>
__global__ void __launch_bounds__(256) quantize64_kernel(const T* __restrict__ x, int64_t n, int64_t n_groups,
                                                         qlrt_codebook4 cb, uint32_t* __restrict__ codes,
                                                         float* __restrict__ absmax,
                                                         unsigned long long* __restrict__ first_bad) {
  __shared__ BinTables t;
  build_bin_tables(t, cb);
  __syncthreads();
  const unsigned pad = (unsigned)cb.pad_code;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  using V = typename AccT<T>::type;
  // warp-uniform trip count: every lane reaches the shuffles
  for (int64_t gb = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); gb < n_groups; gb += stride) {
    const int64_t g = gb + lane;
    const bool act = g < n_groups;  // n_groups % 8 == 0: 8-lane groups are all-in or all-out
    const int64_t i0 = g * 8;
    V v[8];
    if (act) {
      load8<T>(x, i0, n, v);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (V)0;
    }
    V m = (V)0;
    bool finite = true;
    if constexpr (sizeof(V) == 4) {
      // integer max of the magnitude bits: equals the float max for finite
      // values and flags inf/NaN (exponent all ones) in one compare
      unsigned mb = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) mb = max(mb, __float_as_uint(v[j]) & 0x7FFFFFFFu);
      finite = mb < 0x7F800000u;
      m = __uint_as_float(mb);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        finite &= finite_v(v[j]);
        m = fmax(m, fabs(v[j]));
      }
    }
    if (!finite) {
      unsigned long long bad = ~0ull;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (!finite_v(v[j]) && i0 + j < n) bad = min(bad, (unsigned long long)(i0 + j));
      atomicMin(first_bad, bad);
    }
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 2));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 4));
    if (!act) continue;
    const float c = to_f32_const(m);  // f32(absmax) (blockquant.py:166)
    uint32_t word = 0;
    if (c > 0.0f) {
      const float r = __frcp_rn(c);
      const bool fast_ok = r <= 3.402823466e38f;  // subnormal c: 1/c overflows
      if (fast_ok && i0 + 8 <= n) {
#pragma unroll
        for (int j = 0; j < 8; ++j) word |= bin_code(v[j], r, c, t) << (4 * j);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          unsigned k = pad;
          if (i0 + j < n) k = fast_ok ? bin_code(v[j], r, c, t) : exact_code_t((double)v[j], c, t);
          word |= k << (4 * j);
        }
      }
    } else {
      word = pad * 0x11111111u;
    }
    codes[g] = word;
    if ((threadIdx.x & 7) == 0) absmax[g >> 3] = c;
  }
}

// Generic blocksize: absmax per block (one warp per block) ...
template <typename T>
__global__ void absmax_generic_kernel(const T* __restrict__ x, int64_t n, int bs, int64_t nb,
                                      float* __restrict__ absmax,
                                      unsigned long long* __restrict__ first_bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp; b < nb; b += nwarps) {
    double m = 0.0;
    unsigned long long bad = ~0ull;
    for (int64_t i = b * bs + lane; i < min((b + 1) * bs, n); i += 32) {
      double a = fabs((double)x[i]);
      if (!(a <= 1.7976931348623157e308)) bad = min(bad, (unsigned long long)i);
      m = fmax(m, a);
    }
    for (int o = 16; o > 0; o >>= 1) {
      m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    }
    if (lane == 0) {
      absmax[b] = __double2float_rn(m);
      if (bad != ~0ull) atomicMin(first_bad, bad);
    }
  }
}

// ... then one thread per packed byte (two elements, possibly two blocks).
template <typename T>
__global__ void codes_generic_kernel(const T* __restrict__ x, int64_t n, int bs, int64_t n_pad,
                                     qlrt_codebook4 cb, const float* __restrict__ absmax,
                                     uint8_t* __restrict__ codes) {
  __shared__ CodeTables t;
  if (threadIdx.x < 16) {
    t.lo[threadIdx.x] = cb.lo[threadIdx.x];
    t.hi[threadIdx.x] = cb.hi[threadIdx.x];
    if (threadIdx.x < 15) t.mids[threadIdx.x] = cb.mids[threadIdx.x];
  }
  if (threadIdx.x == 0) t.n_mids = cb.n_mids;
  __syncthreads();
  const int64_t nbytes = (n_pad + 1) / 2;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbytes;
       b += (int64_t)gridDim.x * blockDim.x) {
    unsigned byte = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int64_t i = 2 * b + h;
      unsigned k = 0;  // odd tail nibble of pack_codes is 0
      if (i < n_pad) {
        float c = absmax[i / bs];
        if (i < n && c > 0.0f) {
          float r = __frcp_rn(c);
          const double xd = (double)x[i];
          k = (r <= 3.402823466e38f) ? fast_code(xd, r, c, t) : exact_code(xd, c, t);
        } else {
          k = (unsigned)cb.pad_code;
        }
      }
      byte |= k << (4 * h);
    }
    codes[b] = (uint8_t)byte;
  }
}

// ---------------------------------------------------------------------------
// double quantization (doublequant.py:148-187)
// ---------------------------------------------------------------------------

// numpy pairwise_sum (loops_utils.h.src) of float32 values widened to fp64,
// for the (at most one) partial 8192-chunk.  The recursion
//   n <  8   : sequential;   n <= 128 : 8 strided accumulators + tail;
//   otherwise: split at n/2 - (n/2 % 8), left + right
// runs on an explicit stack (no device recursion / dynamic stack).
__device__ double pairwise_leaf(const float* a, int n) {
  if (n < 8) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, (double)a[i]);
    return s;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = (double)a[j];
  const int m = n - n % 8;
  for (int i = 8; i < m; i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], (double)a[i + j]);
  double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (int i = m; i < n; ++i) s = __dadd_rn(s, (double)a[i]);
  return s;
}

// One CTA (512 threads) per 8192-constant buffer chunk.  A full chunk is a
// perfect pairwise tree of 64 leaves of 128; leaf accumulator j of leaf L is
// a[128L + j] + a[128L + j + 8] + ... (16 terms, in order) -- one thread each
// -- and the 8 accumulators combine as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// by xor-shuffles (IEEE addition is commutative, so both partners hold the
// same value).  The encode kernel adds the chunk sums in order from 0.0
// (doublequant.py:164-166).  PDL dependent of phase A.
__global__ void __launch_bounds__(512) dq_chunk_sums_kernel(const float* __restrict__ c, int64_t nb,
                                                            double* __restrict__ chunk_sums) {
  __shared__ double leaf[64];
  asm volatile("griddepcontrol.wait;" ::: "memory");  // phase A's constants
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t base = (int64_t)blockIdx.x * 8192;
  const int len = (int)min((int64_t)8192, nb - base);
  if (len < 8192) {
    // partial chunk: the same recursion tree (split at n/2 - n/2 % 8 down to
    // leaves <= 128), built by thread 0 in preorder, leaves summed in
    // parallel, interior nodes combined children-first (reverse preorder)
    __shared__ int nd_off[256], nd_len[256], nd_l[256], nd_r[256], nd_leaf[256];
    __shared__ double nd_val[256];
    __shared__ int n_nodes, n_leaves;
    if (threadIdx.x == 0) {
      int stack[32], sp = 0, nn = 0, nl = 0;
      nd_off[0] = 0;
      nd_len[0] = len;
      nn = 1;
      stack[sp++] = 0;
      while (sp) {
        const int v = stack[--sp];
        const int L = nd_len[v];
        if (L <= 128) {
          nd_l[v] = nd_r[v] = -1;
          nd_leaf[nl++] = v;
          continue;
        }
        int h = L / 2;
        h -= h % 8;
        const int a = nn++, b = nn++;
        nd_off[a] = nd_off[v];
        nd_len[a] = h;
        nd_off[b] = nd_off[v] + h;
        nd_len[b] = L - h;
        nd_l[v] = a;
        nd_r[v] = b;
        stack[sp++] = b;  // (order of evaluation is irrelevant: values combine by the tree)
        stack[sp++] = a;
      }
      n_nodes = nn;
      n_leaves = nl;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_leaves; i += blockDim.x) {
      const int v = nd_leaf[i];
      nd_val[v] = pairwise_leaf(c + base + nd_off[v], nd_len[v]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int v = n_nodes - 1; v >= 0; --v)  // children have larger indices than their parent
        if (nd_l[v] >= 0) nd_val[v] = __dadd_rn(nd_val[nd_l[v]], nd_val[nd_r[v]]);
      chunk_sums[blockIdx.x] = nd_val[0];
    }
  } else {
    const int L = threadIdx.x >> 3, j = threadIdx.x & 7;
    const float* a = c + base + L * 128 + j;
    float w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = __ldg(a + 8 * i);
    double r = (double)w[0];
#pragma unroll
    for (int i = 1; i < 16; ++i) r = __dadd_rn(r, (double)w[i]);
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (j == 0) leaf[L] = r;
    __syncthreads();
    for (int w2 = 32; w2 >= 1; w2 >>= 1) {
      double sv = 0.0;
      if (threadIdx.x < w2) sv = __dadd_rn(leaf[2 * threadIdx.x], leaf[2 * threadIdx.x + 1]);
      __syncthreads();
      if (threadIdx.x < w2) leaf[threadIdx.x] = sv;
      __syncthreads();
    }
    if (threadIdx.x == 0) chunk_sums[blockIdx.x] = leaf[0];
  }
}


// Persistent: every CTA adds the chunk sums in order (from 0.0) into
// mu = f32(sum / nb) (CTA 0 stores it), then loops over second-level blocks:
// centring by mu, fp64 absmax, c1 = f32(A / max), codes = encode(centered /
// f64(c1))  (doublequant.py:164-186).  PDL dependent of the chunk sums.
__global__ void __launch_bounds__(256) dq_encode_kernel(const float* __restrict__ c, int64_t nb,
                                                        int bs2, const double* __restrict__ chunk_sums,
                                                        int n_chunks, qlrt_fp8spec sp, float* __restrict__ mu_out,
                                                        float* __restrict__ c1,
                                                        uint8_t* __restrict__ codes) {
  __shared__ double s_red[8];
  __shared__ double cs[512];
  __shared__ float s_mu;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  double acc = 0.0;
  for (int b = 0; b < n_chunks; b += 512) {
    __syncthreads();
    for (int i = threadIdx.x; i < 512 && b + i < n_chunks; i += blockDim.x) cs[i] = __ldcg(chunk_sums + b + i);
    __syncthreads();
    if (threadIdx.x == 0) {
      const int e = min(512, n_chunks - b);
      for (int i = 0; i < e; ++i) acc = __dadd_rn(acc, cs[i]);
    }
  }
  if (threadIdx.x == 0) {
    s_mu = __double2float_rn(__ddiv_rn(acc, (double)nb));
    if (blockIdx.x == 0) *mu_out = s_mu;
  }
  __syncthreads();
  const double mu = (double)s_mu;
  const double maxv = fp8_max_value(sp.exp_bits, sp.mant_bits, sp.bias);
  const int64_t n2 = (nb + bs2 - 1) / bs2;
  for (int64_t blk = blockIdx.x; blk < n2; blk += gridDim.x) {
    const int64_t b0 = blk * bs2;
    const int64_t b1 = min(b0 + bs2, nb);
    double amax = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x)
      amax = fmax(amax, fabs(__dsub_rn((double)c[i], mu)));
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    __syncthreads();  // (s_red of the previous block consumed)
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = amax;
    __syncthreads();
    amax = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) amax = fmax(amax, s_red[w]);
    float scale = 0.0f;
    if (amax > 0.0) scale = __double2float_rn(__ddiv_rn(amax, maxv));
    if (threadIdx.x == 0) c1[blk] = scale;  // 0 for flat / underflowing blocks
    const double sd = (double)scale;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      unsigned code = 0u;
      if (scale != 0.0f)
        code = fp8_encode(__ddiv_rn(__dsub_rn((double)c[i], mu), sd), sp.exp_bits, sp.mant_bits, sp.bias, maxv);
      codes[i] = (uint8_t)code;
    }
  }
}

// The same encode with one warp per second-level block (warp-shuffle absmax,
// no block barriers inside the loop, the block's elements spread over the
// lanes): the groups of a call run in parallel across every resident warp.
__global__ void __launch_bounds__(256) dq_encode_warp_kernel(const float* __restrict__ c, int64_t nb, int bs2,
                                                             const double* __restrict__ chunk_sums, int n_chunks,
                                                             qlrt_fp8spec sp, float* __restrict__ mu_out,
                                                             float* __restrict__ c1, uint8_t* __restrict__ codes) {
  __shared__ double cs[512];
  __shared__ float s_mu;
  // The first block's constants go to registers before the wait: this grid
  // starts only after the chunk-sum grid passed its own wait (its trigger
  // follows it), i.e. after the producer of c completed -- only the chunk
  // sums need the wait.  Saves a dependent round trip and the second read.
  constexpr int PRE = 8;  // blocksize2 <= 256
  const int lane = threadIdx.x & 31;
  const int64_t n2 = (nb + bs2 - 1) / bs2;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t blk_first = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const bool pre = bs2 <= 32 * PRE && blk_first < n2;
  float pv[PRE];
#pragma unroll
  for (int k = 0; k < PRE; ++k) pv[k] = 0.0f;
  if (pre) {
    const int64_t b0 = blk_first * bs2, b1 = min(b0 + bs2, nb);
#pragma unroll
    for (int k = 0; k < PRE; ++k)
      if (b0 + lane + 32 * k < b1) pv[k] = __ldg(c + b0 + lane + 32 * k);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  double acc = 0.0;
  for (int b = 0; b < n_chunks; b += 512) {
    __syncthreads();
    for (int i = threadIdx.x; i < 512 && b + i < n_chunks; i += blockDim.x) cs[i] = __ldcg(chunk_sums + b + i);
    __syncthreads();
    if (threadIdx.x == 0) {
      const int e = min(512, n_chunks - b);
      for (int i = 0; i < e; ++i) acc = __dadd_rn(acc, cs[i]);
    }
  }
  if (threadIdx.x == 0) {
    s_mu = __double2float_rn(__ddiv_rn(acc, (double)nb));
    if (blockIdx.x == 0) *mu_out = s_mu;
  }
  __syncthreads();
  const double mu = (double)s_mu;
  const double maxv = fp8_max_value(sp.exp_bits, sp.mant_bits, sp.bias);
  for (int64_t blk = blk_first; blk < n2; blk += warps) {
    const int64_t b0 = blk * bs2;
    const int64_t b1 = min(b0 + bs2, nb);
    const bool in_regs = pre && blk == blk_first;
    double amax = 0.0;
    if (in_regs) {
#pragma unroll
      for (int k = 0; k < PRE; ++k)
        if (b0 + lane + 32 * k < b1) amax = fmax(amax, fabs(__dsub_rn((double)pv[k], mu)));
    } else {
      for (int64_t i = b0 + lane; i < b1; i += 32) amax = fmax(amax, fabs(__dsub_rn((double)__ldg(c + i), mu)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    float scale = 0.0f;
    if (amax > 0.0) scale = __double2float_rn(__ddiv_rn(amax, maxv));
    if (lane == 0) c1[blk] = scale;  // 0 for flat / underflowing blocks
    const double sd = (double)scale;
    if (in_regs) {
#pragma unroll
      for (int k = 0; k < PRE; ++k) {
        const int64_t i = b0 + lane + 32 * k;
        if (i >= b1) break;
        unsigned code = 0u;
        if (scale != 0.0f)
          code = fp8_encode(__ddiv_rn(__dsub_rn((double)pv[k], mu), sd), sp.exp_bits, sp.mant_bits, sp.bias, maxv);
        codes[i] = (uint8_t)code;
      }
    } else {
      for (int64_t i = b0 + lane; i < b1; i += 32) {
        unsigned code = 0u;
        if (scale != 0.0f)
          code = fp8_encode(__ddiv_rn(__dsub_rn((double)__ldg(c + i), mu), sd), sp.exp_bits, sp.mant_bits, sp.bias,
                            maxv);
        codes[i] = (uint8_t)code;
      }
    }
  }
}

__global__ void dq_decompress_kernel(const uint8_t* __restrict__ codes,
                                     const float* __restrict__ c1, const float* __restrict__ mu,
                                     int64_t nb, int bs2, qlrt_fp8spec sp,
                                     float* __restrict__ out) {
  const float m = *mu;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = dq_constant(codes[i], c1[i / bs2], m, sp);
}

// ---------------------------------------------------------------------------
// dequantize (blockquant.py:198-213): out = f32(values[code] * f64(c)).
// blocksize 64 fast path: a warp owns 32 consecutive 64-blocks, one per lane.
// Each lane loads its 32 code bytes (two 16B loads) with its DQ byte and c1,
// computes the block's 16 exact products f64(v_i) * f64(c) once (16 DMUL) into
// its column of a [code][thread] shared table (conflict-free reads), decodes
// its block into a 128B-swizzled row of a per-warp staging buffer, and the
// warp then writes the 32 rows out with fully coalesced 16B stores.
// ---------------------------------------------------------------------------
constexpr int DQ_TPB = 128;  // threads per CTA of the dequant kernel

// 4 codes (nibbles of the low 16 bits of w) -> 4 bf16 from a 16-entry table
// held as lo/hi byte planes: 3 byte-permutes per plane (codes 0-7 / 8-15 and
// a select on bit 3), 2 to interleave -- no shared-memory table reads.
__device__ __forceinline__ void lookup4_bf16(uint32_t w, const uint32_t (&L)[4], const uint32_t (&H)[4],
                                             uint32_t& o0, uint32_t& o1) {
  const uint32_t sel = w & 0x7777u;
  const uint32_t bsel = ((w >> 1) & 0x4444u) | 0x3210u;
  const uint32_t lo = __byte_perm(__byte_perm(L[0], L[1], sel), __byte_perm(L[2], L[3], sel), bsel);
  const uint32_t hi = __byte_perm(__byte_perm(H[0], H[1], sel), __byte_perm(H[2], H[3], sel), bsel);
  o0 = __byte_perm(lo, hi, 0x5140);
  o1 = __byte_perm(lo, hi, 0x7362);
}

template <int OUT>
__global__ void __launch_bounds__(DQ_TPB) dequant64_kernel(const uint4* __restrict__ codes, int64_t n, qlrt_codebook4 cb,
                                                        const float* __restrict__ absmax,
                                                        const uint8_t* __restrict__ dq_codes,
                                                        const float* __restrict__ c1, const float* __restrict__ mu,
                                                        int bs2, qlrt_fp8spec sp, void* __restrict__ out) {
  using LT = typename std::conditional<OUT == QLRT_F64, double, float>::type;
  using OT = typename std::conditional<OUT == QLRT_F64, double,
                                       typename std::conditional<OUT == QLRT_F32, float, __nv_bfloat16>::type>::type;
  constexpr int EPP = 128 / sizeof(OT);     // elements per lane per pass (one 128B row)
  constexpr int PASSES = 64 / EPP;          // 1 (bf16), 2 (f32), 4 (f64)
  __shared__ LT lut[16 * DQ_TPB];
  __shared__ __align__(16) uint8_t stage[DQ_TPB / 32][32 * 128];
  const float mu_v = dq_codes ? *mu : 0.0f;
  const int64_t nb = cdiv(n, 64);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  LT* col = lut + threadIdx.x;
  uint8_t* st = stage[wid];
  const int64_t n_warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t wb = ((int64_t)blockIdx.x * (blockDim.x >> 5) + wid) * 32; wb < nb; wb += n_warps_total * 32) {
    const int64_t blk = wb + lane;
    const bool live = blk < nb;
    uint4 w0 = make_uint4(0, 0, 0, 0), w1 = w0;
    float c = 0.0f;
    if (live) {
      w0 = __ldg(codes + 2 * blk);
      w1 = __ldg(codes + 2 * blk + 1);
      c = dq_codes ? dq_constant(__ldg(dq_codes + blk), __ldg(c1 + blk / bs2), mu_v, sp) : __ldg(absmax + blk);
    }
    const double cd = (double)c;
    uint32_t Lp[4], Hp[4];  // bf16 path: exact table bf16(f32(v64*c64)) as lo/hi byte planes
    if constexpr (OUT == QLRT_BF16) {
      uint32_t P[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        P[j] = pack_bf16x2(__double2float_rn(__dmul_rn(cb.values[2 * j], cd)),
                           __double2float_rn(__dmul_rn(cb.values[2 * j + 1], cd)));
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        Lp[q] = __byte_perm(P[2 * q], P[2 * q + 1], 0x6420);
        Hp[q] = __byte_perm(P[2 * q], P[2 * q + 1], 0x7531);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const double d = __dmul_rn(cb.values[i], cd);
        if constexpr (OUT == QLRT_F64) col[i * DQ_TPB] = d;
        else col[i * DQ_TPB] = __double2float_rn(d);
      }
    }
    const uint32_t ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
    for (int pass = 0; pass < PASSES; ++pass) {
      // this lane's row: elements [pass*EPP, (pass+1)*EPP) of its block, 8 x 16B chunks
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        constexpr int EPC = 16 / sizeof(OT);  // elements per 16B chunk
        uint32_t pk[4];
        if constexpr (OUT == QLRT_BF16) {
          const uint32_t w = ws[pass * 8 + ch];  // 8 codes -> 8 bf16 by register byte-permutes
          lookup4_bf16(w, Lp, Hp, pk[0], pk[1]);
          lookup4_bf16(w >> 16, Lp, Hp, pk[2], pk[3]);
        } else {
          const int e = pass * EPP + ch * EPC;  // first element of the chunk
          const uint32_t w = ws[e >> 3] >> (4 * (e & 7));
          LT v[EPC];
#pragma unroll
          for (int j = 0; j < EPC; ++j) v[j] = col[((w >> (4 * j)) & 15u) * DQ_TPB];
          const uint4 u = *reinterpret_cast<const uint4*>(v);
          pk[0] = u.x; pk[1] = u.y; pk[2] = u.z; pk[3] = u.w;
        }
        *reinterpret_cast<uint4*>(st + lane * 128 + ((ch ^ (lane & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      __syncwarp();
      // coalesced copy-out: 4 rows (blocks) x 128B per instruction
      if (wb + 32 <= nb && (wb + 32) * 64 <= n) {  // whole warp in range: no per-store checks
        uint8_t* ob = reinterpret_cast<uint8_t*>(static_cast<OT*>(out) + wb * 64 + pass * EPP);
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int row = it * 4 + (lane >> 3), ch = lane & 7;
          const uint4 u = *reinterpret_cast<const uint4*>(st + row * 128 + ((ch ^ (row & 7)) << 4));
          *reinterpret_cast<uint4*>(ob + row * (64 * (int)sizeof(OT)) + ch * 16) = u;
        }
        __syncwarp();
        continue;
      }
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int row = it * 4 + (lane >> 3), ch = lane & 7;
        const uint4 u = *reinterpret_cast<const uint4*>(st + row * 128 + ((ch ^ (row & 7)) << 4));
        const int64_t b = wb + row;
        const int64_t e0 = b * 64 + pass * EPP + ch * (16 / (int)sizeof(OT));
        if (b < nb) {
          OT* o = static_cast<OT*>(out) + e0;
          if (e0 + 16 / (int)sizeof(OT) <= n) {
            *reinterpret_cast<uint4*>(o) = u;
          } else {
            const OT* e = reinterpret_cast<const OT*>(&u);
            for (int j = 0; j < 16 / (int)sizeof(OT) && e0 + j < n; ++j) o[j] = e[j];
          }
        }
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// bf16 output, blocksize 64, no shared-memory staging: one lane per 64-block.
// A lane loads its block's 32 code bytes with one 256-bit load (a warp reads
// 1 KB contiguous), builds the block's 16-entry table bf16(f32(f64(v_i) *
// f64(c))) exactly (16 DMUL with the codebook as constant-bank operands), split
// into lo/hi byte planes, decodes 8 codes per 21 integer ops (lookup8_bf16) and
// writes its 128 output bytes with four 256-bit stores.  The DQ constant comes
// from a 256-entry fp64 decode table of the 8-bit float in shared memory.
// Each warp owns a balanced contiguous range of 32-block steps and prefetches
// step i+1's codes and constants before decoding step i.
// ---------------------------------------------------------------------------
constexpr int DQB_TPB = 256;

__device__ __forceinline__ void st_global_v8(void* p, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                             uint32_t a4, uint32_t a5, uint32_t a6, uint32_t a7) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a0), "r"(a1),
               "r"(a2), "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7)
               : "memory");
}

__device__ __forceinline__ void ld_stream_v8(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}

// 8 codes (nibbles of w, element order) -> 8 bf16 in o[0..3]
__device__ __forceinline__ void lookup8_bf16(uint32_t w, const uint32_t (&L)[4], const uint32_t (&H)[4],
                                             uint32_t& o0, uint32_t& o1, uint32_t& o2, uint32_t& o3) {
  const uint32_t sel = w & 0x77777777u;
  const uint32_t bs = ((w >> 1) & 0x44444444u) | 0x32103210u;
  const uint32_t selh = sel >> 16, bsh = bs >> 16;
  const uint32_t la = __byte_perm(__byte_perm(L[0], L[1], sel), __byte_perm(L[2], L[3], sel), bs);
  const uint32_t ha = __byte_perm(__byte_perm(H[0], H[1], sel), __byte_perm(H[2], H[3], sel), bs);
  const uint32_t lb = __byte_perm(__byte_perm(L[0], L[1], selh), __byte_perm(L[2], L[3], selh), bsh);
  const uint32_t hb = __byte_perm(__byte_perm(H[0], H[1], selh), __byte_perm(H[2], H[3], selh), bsh);
  o0 = __byte_perm(la, ha, 0x5140);
  o1 = __byte_perm(la, ha, 0x7362);
  o2 = __byte_perm(lb, hb, 0x5140);
  o3 = __byte_perm(lb, hb, 0x7362);
}

template <bool DQ>
#ifndef QLRT_DQB_MINB
#define QLRT_DQB_MINB 4  // 4 resident CTAs per SM (64 regs, no spills): C1 +7.7% over 3
#endif
__global__ void __launch_bounds__(DQB_TPB, QLRT_DQB_MINB) dequant64_bf16_kernel(const uint8_t* __restrict__ codes, int64_t n,
                                                                    qlrt_codebook4 cb,
                                                                    const float* __restrict__ absmax,
                                                                    const uint8_t* __restrict__ dq_codes,
                                                                    const float* __restrict__ c1,
                                                                    const float* __restrict__ mu, int bs2_shift,
                                                                    qlrt_fp8spec sp, __nv_bfloat16* __restrict__ out) {
  __shared__ double fp8_lut[256];
  const int lane = threadIdx.x & 31;
  const int64_t nb = cdiv(n, 64), n_steps = cdiv(nb, 32);
  const int64_t n_warps = (int64_t)gridDim.x * (DQB_TPB / 32);
  const int64_t w = (int64_t)blockIdx.x * (DQB_TPB / 32) + (threadIdx.x >> 5);
  const int64_t s_beg = n_steps * w / n_warps, s_end = n_steps * (w + 1) / n_warps;

  // PDL: the next launch may start its prologue as this grid drains; our
  // reads wait for the predecessor grid (a no-op without the attribute)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (DQ) fp8_lut[threadIdx.x] = fp8_decode_fast(threadIdx.x, sp);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  uint32_t cw[8];
  float craw = 0.0f;   // absmax, or c1 of the block (DQ)
  uint32_t dqb = 0;    // DQ code byte
  auto fetch = [&](int64_t s) {
    const int64_t blk = s * 32 + lane;
    if (blk < nb) {
      ld_stream_v8(codes + blk * 32, cw);
      if (DQ) {
        dqb = __ldg(dq_codes + blk);
        craw = __ldg(c1 + (blk >> bs2_shift));
      } else {
        craw = __ldg(absmax + blk);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) cw[i] = 0u;
    }
  };
  if (s_beg < s_end) fetch(s_beg);
  if (DQ) __syncthreads();  // (the fp8 table)
  const double mu_d = DQ ? (double)__ldg(mu) : 0.0;
  for (int64_t s = s_beg; s < s_end; ++s) {
    uint32_t cur[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) cur[i] = cw[i];
    float c;
    if (DQ) {
      const double r = __dadd_rn(__dmul_rn(fp8_lut[dqb], (double)craw), mu_d);
      c = __double2float_rn(r > 0.0 ? r : 0.0);
    } else {
      c = craw;
    }
    if (s + 1 < s_end) fetch(s + 1);
    const double cd = (double)c;
    uint32_t L[4], H[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t p0 = pack_bf16x2(__double2float_rn(__dmul_rn(cb.values[4 * q], cd)),
                                      __double2float_rn(__dmul_rn(cb.values[4 * q + 1], cd)));
      const uint32_t p1 = pack_bf16x2(__double2float_rn(__dmul_rn(cb.values[4 * q + 2], cd)),
                                      __double2float_rn(__dmul_rn(cb.values[4 * q + 3], cd)));
      L[q] = __byte_perm(p0, p1, 0x6420);
      H[q] = __byte_perm(p0, p1, 0x7531);
    }
    const int64_t blk = s * 32 + lane;
    __nv_bfloat16* dst = out + blk * 64;
    if (blk * 64 + 64 <= n) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t o[8];
        lookup8_bf16(cur[2 * j], L, H, o[0], o[1], o[2], o[3]);
        lookup8_bf16(cur[2 * j + 1], L, H, o[4], o[5], o[6], o[7]);
        st_global_v8(dst + 16 * j, o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]);
      }
    } else if (blk < nb) {  // ragged last block: element-wise, registers only
      unsigned short* d16 = reinterpret_cast<unsigned short*>(dst);
      const int rem = (int)(n - blk * 64);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t o[4];
        lookup8_bf16(cur[j], L, H, o[0], o[1], o[2], o[3]);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (8 * j + e < rem) d16[8 * j + e] = (unsigned short)((e & 1) ? (o[e >> 1] >> 16) : (o[e >> 1] & 0xFFFFu));
      }
    }
  }
}

// generic blocksize: one thread per element
template <int OUT>
__global__ void dequant_generic_kernel(const uint8_t* __restrict__ codes, int64_t n, int bs,
                                       qlrt_codebook4 cb, const float* __restrict__ absmax,
                                       const uint8_t* __restrict__ dq_codes,
                                       const float* __restrict__ c1, const float* __restrict__ mu,
                                       int bs2, qlrt_fp8spec sp, void* __restrict__ out) {
  __shared__ double vals[16];
  if (threadIdx.x < 16) vals[threadIdx.x] = cb.values[threadIdx.x];
  __syncthreads();
  const float mu_v = dq_codes ? *mu : 0.0f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = i / bs;
    float c = dq_codes ? dq_constant(dq_codes[blk], c1[blk / bs2], mu_v, sp) : absmax[blk];
    unsigned code = (codes[i >> 1] >> (4 * (i & 1))) & 15u;
    const double d = __dmul_rn(vals[code], (double)c);
    if (OUT == QLRT_F64) static_cast<double*>(out)[i] = d;
    else if (OUT == QLRT_BF16) static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(__double2float_rn(d));
    else static_cast<float*>(out)[i] = __double2float_rn(d);
  }
}

__global__ void fp8_encode_kernel(const double* __restrict__ x, int64_t n, qlrt_fp8spec sp,
                                  uint8_t* __restrict__ out) {
  const double maxv = fp8_max_value(sp.exp_bits, sp.mant_bits, sp.bias);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint8_t)fp8_encode(x[i], sp.exp_bits, sp.mant_bits, sp.bias, maxv);
}

__global__ void fp8_decode_kernel(const uint8_t* __restrict__ c, int64_t n, qlrt_fp8spec sp,
                                  double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = fp8_decode(c[i], sp.exp_bits, sp.mant_bits, sp.bias);
}

__global__ void pack4_kernel(const uint8_t* __restrict__ codes, int64_t count,
                             uint8_t* __restrict__ packed) {
  const int64_t nbytes = (count + 1) / 2;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbytes;
       b += (int64_t)gridDim.x * blockDim.x) {
    unsigned lo = codes[2 * b] & 15u;
    unsigned hi = (2 * b + 1 < count) ? (codes[2 * b + 1] & 15u) : 0u;
    packed[b] = (uint8_t)(lo | (hi << 4));
  }
}

__global__ void unpack4_kernel(const uint8_t* __restrict__ packed, int64_t count,
                               uint8_t* __restrict__ codes) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    codes[i] = (packed[i >> 1] >> (4 * (i & 1))) & 15u;
}

static inline int grid_for(int64_t work, int threads, int per_sm = 8) {
  int64_t g = cdiv(work, threads);
  int64_t cap = (int64_t)kNumSMs * per_sm;
  return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

}  // namespace qlrt

using namespace qlrt;

extern "C" {

qlrt_status qlrt_quantize4(const void* x, int x_dtype, int64_t n, int blocksize,
                           const qlrt_codebook4* cb, uint8_t* codes, float* absmax,
                           int64_t* first_bad, void* stream) {
  if (n <= 0 || blocksize < 1 || !cb || !x || !codes || !absmax || !first_bad) return QLRT_ERR_ARG;
  if (x_dtype != QLRT_F32 && x_dtype != QLRT_BF16 && x_dtype != QLRT_F64) return QLRT_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nb = cdiv(n, blocksize);
  // sentinel 0x7F7F...7F (> any index); memset is graph-capturable
  if (cudaMemsetAsync(first_bad, 0x7F, 8, s) != cudaSuccess) return QLRT_ERR_CUDA;
  auto* fb = reinterpret_cast<unsigned long long*>(first_bad);
  const bool aligned = (((uintptr_t)x) & 15) == 0 && (((uintptr_t)codes) & 3) == 0;
  const bool aligned32 = (((uintptr_t)x) & 31) == 0 && (((uintptr_t)codes) & 3) == 0;
  if (blocksize == 64 && n % 64 == 0 && aligned32 && (x_dtype == QLRT_F32 || x_dtype == QLRT_BF16)) {
    const int64_t n_groups = nb * 8;
    const int64_t want = cdiv(n_groups, 256);
    const int grid = (int)(want < (int64_t)kNumSMs * QLRT_Q_MINB ? want : (int64_t)kNumSMs * QLRT_Q_MINB);  // resident
    constexpr int psm = PBIN * 32 * 8;  // private-column bin table
    // (no PDL attribute: the first-bad sentinel memset precedes it)
    cudaLaunchConfig_t cfg{};
    cfg.stream = s;
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = psm;
    const cudaError_t e =
        x_dtype == QLRT_F32
            ? cudaLaunchKernelEx(&cfg, quantize64_stream_kernel<float>, (const float*)x, n_groups, *cb,
                                 (uint32_t*)codes, absmax, fb)
            : cudaLaunchKernelEx(&cfg, quantize64_stream_kernel<__nv_bfloat16>, (const __nv_bfloat16*)x, n_groups,
                                 *cb, (uint32_t*)codes, absmax, fb);
    if (e != cudaSuccess) return QLRT_ERR_CUDA;
  } else if (blocksize == 64 && aligned) {
    const int64_t n_groups = nb * 8;
    const int grid = grid_for(n_groups, 256, 8);
    if (x_dtype == QLRT_F32)
      quantize64_kernel<float><<<grid, 256, 0, s>>>((const float*)x, n, n_groups, *cb, (uint32_t*)codes, absmax, fb);
    else if (x_dtype == QLRT_BF16)
      quantize64_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)x, n, n_groups, *cb,
                                                            (uint32_t*)codes, absmax, fb);
    else
      quantize64_kernel<double><<<grid, 256, 0, s>>>((const double*)x, n, n_groups, *cb, (uint32_t*)codes, absmax, fb);
  } else {
    const int ga = grid_for(nb * 32, 256, 8);
    const int gc = grid_for(cdiv(nb * blocksize, 2), 256, 8);
    if (x_dtype == QLRT_F32) {
      absmax_generic_kernel<float><<<ga, 256, 0, s>>>((const float*)x, n, blocksize, nb, absmax, fb);
      codes_generic_kernel<float><<<gc, 256, 0, s>>>((const float*)x, n, blocksize, nb * blocksize, *cb, absmax, codes);
    } else if (x_dtype == QLRT_BF16) {
      absmax_generic_kernel<__nv_bfloat16><<<ga, 256, 0, s>>>((const __nv_bfloat16*)x, n, blocksize, nb, absmax, fb);
      codes_generic_kernel<__nv_bfloat16><<<gc, 256, 0, s>>>((const __nv_bfloat16*)x, n, blocksize, nb * blocksize,
                                                             *cb, absmax, codes);
    } else {
      absmax_generic_kernel<double><<<ga, 256, 0, s>>>((const double*)x, n, blocksize, nb, absmax, fb);
      codes_generic_kernel<double><<<gc, 256, 0, s>>>((const double*)x, n, blocksize, nb * blocksize, *cb, absmax,
                                                      codes);
    }
  }
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

// chunk sums of the DQ mean (fp64 per 8192-constant chunk)
size_t qlrt_dq_workspace_bytes(int64_t nb) { return (size_t)cdiv(nb, 8192) * sizeof(double) + 16; }

qlrt_status qlrt_dq_compress(const float* absmax, int64_t nb, int blocksize2, qlrt_fp8spec spec,
                             void* workspace, float* mu, float* c1, uint8_t* dq_codes,
                             void* stream) {
  if (nb <= 0 || blocksize2 < 1 || !absmax || !workspace || !mu || !c1 || !dq_codes)
    return QLRT_ERR_ARG;
  if (spec.exp_bits + spec.mant_bits != 7 || spec.exp_bits < 1 || spec.bias < 0) return QLRT_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n_chunks = cdiv(nb, 8192);
  double* sums = (double*)workspace;
  // chunk sums, then the persistent encode (each CTA adds the chunk sums in
  // order itself: no ticket, no memset), both PDL-chained to their producer
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = policy(P_PDL) ? 1 : 0;
  cfg.stream = s;
  cfg.gridDim = dim3((unsigned)n_chunks);
  cfg.blockDim = dim3(512);
  if (cudaLaunchKernelEx(&cfg, dq_chunk_sums_kernel, absmax, nb, sums) != cudaSuccess) return QLRT_ERR_CUDA;
  const int64_t n2 = cdiv(nb, blocksize2);
  cfg.blockDim = dim3(256);
  if (blocksize2 <= 4096) {  // one warp per second-level block
    const int64_t ctas = cdiv(n2, 8);
    cfg.gridDim = dim3((unsigned)(ctas < (int64_t)kNumSMs * 8 ? ctas : (int64_t)kNumSMs * 8));
    if (cudaLaunchKernelEx(&cfg, dq_encode_warp_kernel, absmax, nb, blocksize2, (const double*)sums, (int)n_chunks,
                           spec, mu, c1, dq_codes) != cudaSuccess)
      return QLRT_ERR_CUDA;
  } else {
    cfg.gridDim = dim3((unsigned)(n2 < (int64_t)kNumSMs * 8 ? n2 : (int64_t)kNumSMs * 8));
    if (cudaLaunchKernelEx(&cfg, dq_encode_kernel, absmax, nb, blocksize2, (const double*)sums, (int)n_chunks, spec,
                           mu, c1, dq_codes) != cudaSuccess)
      return QLRT_ERR_CUDA;
  }
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_dq_decompress(const uint8_t* dq_codes, const float* c1, const float* mu,
                               int64_t nb, int blocksize2, qlrt_fp8spec spec, float* out,
                               void* stream) {
  if (nb <= 0 || blocksize2 < 1 || !dq_codes || !c1 || !mu || !out) return QLRT_ERR_ARG;
  dq_decompress_kernel<<<grid_for(nb, 256), 256, 0, (cudaStream_t)stream>>>(dq_codes, c1, mu, nb,
                                                                            blocksize2, spec, out);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_dequantize4(const uint8_t* codes, int64_t n, int blocksize,
                             const qlrt_codebook4* cb, const float* absmax,
                             const uint8_t* dq_codes, const float* c1, const float* mu,
                             int blocksize2, qlrt_fp8spec spec, void* out, int out_dtype,
                             void* stream) {
  if (n <= 0 || blocksize < 1 || !codes || !cb || !out) return QLRT_ERR_ARG;
  if (!absmax && !(dq_codes && c1 && mu)) return QLRT_ERR_ARG;
  if (out_dtype != QLRT_F32 && out_dtype != QLRT_BF16 && out_dtype != QLRT_F64) return QLRT_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const bool aligned = (((uintptr_t)codes) & 15) == 0 && (((uintptr_t)out) & 15) == 0;
  const bool pow2_bs2 = blocksize2 > 0 && (blocksize2 & (blocksize2 - 1)) == 0;
  if (blocksize == 64 && out_dtype == QLRT_BF16 && (((uintptr_t)codes) & 31) == 0 &&
      (((uintptr_t)out) & 31) == 0 && (!dq_codes || (pow2_bs2 && (((uintptr_t)dq_codes) & 15) == 0))) {
    // QLRT_DQB_MINB CTAs x 8 warps resident per SM, balanced 32-block steps per warp
    const int64_t ctas = cdiv(cdiv(cdiv(n, 64), 32), DQB_TPB / 32);
    // long streams: 16 CTAs per SM launched (3 resident) -- short-lived CTAs
    // overlap one another's tails and balance dynamically (+13% at the 65B
    // shapes: 6.1 vs 5.4 TB/s); short ones (< 4 steps per warp) stay at one
    // resident wave.  QLRT_DQB_CTAS_PER_SM overrides.
    const int e_g = policy(P_DQB_CTAS_PER_SM);
    const int64_t steps = cdiv(cdiv(n, 64), 32);
    const int64_t per_sm =
        e_g > 0 ? e_g : (steps > 4 * (int64_t)kNumSMs * QLRT_DQB_MINB * (DQB_TPB / 32) ? 16 : QLRT_DQB_MINB);
    const int g = (int)(ctas < (int64_t)kNumSMs * per_sm ? ctas : (int64_t)kNumSMs * per_sm);
    const int sh = pow2_bs2 ? __builtin_ctz((unsigned)blocksize2) : 0;
    // programmatic dependent launch: back-to-back dequantizations overlap one
    // another's launch and prologue with the predecessor's tail
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = policy(P_PDL) ? 1 : 0;
    cfg.stream = s;
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(DQB_TPB);
    const cudaError_t e =
        dq_codes ? cudaLaunchKernelEx(&cfg, dequant64_bf16_kernel<true>, codes, n, *cb, absmax, dq_codes, c1, mu, sh,
                                      spec, (__nv_bfloat16*)out)
                 : cudaLaunchKernelEx(&cfg, dequant64_bf16_kernel<false>, codes, n, *cb, absmax, dq_codes, c1, mu,
                                      sh, spec, (__nv_bfloat16*)out);
    if (e != cudaSuccess) return QLRT_ERR_CUDA;
  } else if (blocksize == 64 && aligned) {
    const int g = grid_for(cdiv(n, 64), DQ_TPB, 16);
#define QLRT_DQ64(O) dequant64_kernel<O><<<g, DQ_TPB, 0, s>>>((const uint4*)codes, n, *cb, absmax, dq_codes, c1, mu, \
                                                           blocksize2, spec, out)
    if (out_dtype == QLRT_BF16) QLRT_DQ64(QLRT_BF16);
    else if (out_dtype == QLRT_F32) QLRT_DQ64(QLRT_F32);
    else QLRT_DQ64(QLRT_F64);
#undef QLRT_DQ64
  } else {
    const int g = grid_for(n, 256, 8);
#define QLRT_DQG(O) dequant_generic_kernel<O><<<g, 256, 0, s>>>(codes, n, blocksize, *cb, absmax, dq_codes, c1, mu, \
                                                                blocksize2, spec, out)
    if (out_dtype == QLRT_BF16) QLRT_DQG(QLRT_BF16);
    else if (out_dtype == QLRT_F32) QLRT_DQG(QLRT_F32);
    else QLRT_DQG(QLRT_F64);
#undef QLRT_DQG
  }
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_fp8_encode(const double* x, int64_t n, qlrt_fp8spec spec, uint8_t* out, void* stream) {
  if (!x || !out || n <= 0 || spec.exp_bits + spec.mant_bits != 7) return QLRT_ERR_ARG;
  fp8_encode_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, n, spec, out);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_fp8_decode(const uint8_t* codes, int64_t n, qlrt_fp8spec spec, double* out, void* stream) {
  if (!codes || !out || n <= 0 || spec.exp_bits + spec.mant_bits != 7) return QLRT_ERR_ARG;
  fp8_decode_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(codes, n, spec, out);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_pack4(const uint8_t* codes, int64_t count, uint8_t* packed, void* stream) {
  if (count <= 0 || !codes || !packed) return QLRT_ERR_ARG;
  pack4_kernel<<<grid_for(cdiv(count, 2), 256), 256, 0, (cudaStream_t)stream>>>(codes, count, packed);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_unpack4(const uint8_t* packed, int64_t count, uint8_t* codes, void* stream) {
  if (count <= 0 || !codes || !packed) return QLRT_ERR_ARG;
  unpack4_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(packed, count, codes);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

const char* qlrt_build_info(void) { return "qlrt_b200 sm_100a"; }

}  // extern "C"
