// Shared helpers for the qlrt_b200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <atomic>
#include "qlrt_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "qlrt_b200 kernels are written for sm_100a (B200) only"
#endif

#define QLRT_CHECK_LAUNCH()                                    \
  do {                                                         \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return QLRT_ERR_CUDA;               \
  } while (0)

namespace qlrt {

constexpr int kNumSMs = 148;

// ---- launch policies ------------------------------------------------------
// Scheduling switches of the engine (measured A/B knobs).  Read
// from the environment ONCE (first use), afterwards only through
// qlrt_set_policy(): no getenv on the launch path.  One process-wide table of
// atomics shared by every translation unit of the library.
enum Policy {
  P_PAIR, P_SIDE, P_TILE512, P_STAGGER, P_TMAOUT, P_HALFTAIL, P_PDL, P_SHARE, P_STREAMK, P_OVERLAP,
  P_OVERLAP_SMS, P_PDL_TRIGGER, P_STREAMK_SKINNY, P_CSPLIT, P_OVERLAP_BWD, P_GEMV_WL, P_DQB_CTAS_PER_SM,
  P_GEMV_MMA, P_DIAG_SKIP, P_CL2, P_SIDE_SMS, P_SKINNY_CTAS, P_GEMV_MIN_UNITS, P_SK512, P_PRIO, P_COUNT
};
struct PolicyDef {
  const char* env;
  int dflt;
};
inline const PolicyDef kPolicies[P_COUNT] = {
    {"QLRT_PAIR", -1},         {"QLRT_SIDE", 1},           {"QLRT_TILE512", 1},   {"QLRT_STAGGER", 0},
    {"QLRT_TMAOUT", 1},        {"QLRT_HALFTAIL", 1},       {"QLRT_PDL", 1},       {"QLRT_SHARE", 0},
    {"QLRT_STREAMK", 1},       {"QLRT_OVERLAP", 1},        {"QLRT_OVERLAP_SMS", 8}, {"QLRT_PDL_TRIGGER", 1},
    {"QLRT_STREAMK_SKINNY", 0}, {"QLRT_CSPLIT", 0},        {"QLRT_OVERLAP_BWD", 0}, {"QLRT_GEMV_WL", -1},
    {"QLRT_DQB_CTAS_PER_SM", -1}, {"QLRT_GEMV_MMA", 1},
    // QLRT_DIAG_SKIP is measurement only: 1 skips dl2/dl1, 2 skips dT (wrong results)
    {"QLRT_DIAG_SKIP", 0},     {"QLRT_CL2", 0},          {"QLRT_SIDE_SMS", 0},     {"QLRT_SKINNY_CTAS", 148}, {"QLRT_GEMV_MIN_UNITS", 8}, {"QLRT_SK512", 0},
    // QLRT_PRIO (measured, off): 1 launches the caller's stream at the
    // device's greatest priority, 2 the side stream (C3: -2.5% / neutral)
    {"QLRT_PRIO", 0}};
constexpr int kPolicyUnset = -0x7fffffff;
inline std::atomic<int> g_policy[P_COUNT];
inline std::atomic<bool> g_policy_init{false};

inline void policy_load_env() {
  for (int i = 0; i < P_COUNT; ++i) {
    const char* e = getenv(kPolicies[i].env);
    g_policy[i].store(e ? atoi(e) : kPolicies[i].dflt, std::memory_order_relaxed);
  }
  g_policy_init.store(true, std::memory_order_release);
}
inline int policy(Policy p) {
  if (!g_policy_init.load(std::memory_order_acquire)) policy_load_env();
  return g_policy[p].load(std::memory_order_relaxed);
}

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// greatest launch priority of the current device (numerically lowest)
inline int high_priority() {
  static std::atomic<int> cached{1};
  int p = cached.load(std::memory_order_relaxed);
  if (p == 1) {
    int lo = 0, hi = 0;
    p = cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess ? hi : 0;
    cached.store(p, std::memory_order_relaxed);
  }
  return p;
}

// ---- 8-bit float of the double quantizer (doublequant.py:33-121) ----------
// decode: exact dyadic value of every byte (no NaN/Inf; 0x80 is -0.0)
__device__ __forceinline__ double fp8_decode(unsigned b, int E, int M, int B) {
  unsigned e = (b >> M) & ((1u << E) - 1u);
  unsigned m = b & ((1u << M) - 1u);
  double mag = (e == 0) ? ldexp((double)m, 1 - B - M)
                        : ldexp((double)((1u << M) + m), (int)e - B - M);
  return (b >> 7) ? -mag : mag;
}

__host__ __device__ inline double fp8_max_value(int E, int M, int B) {
  // (2 - 2^-M) * 2^(2^E - 1 - B)
  double top = 2.0 - 1.0 / (double)(1 << M);
  int ex = (1 << E) - 1 - B;
  double p = 1.0;
  if (ex >= 0) for (int i = 0; i < ex; ++i) p *= 2.0;
  else for (int i = 0; i < -ex; ++i) p *= 0.5;
  return top * p;
}

// encode: nearest grid value, ties away from zero, clamp at +-max
// (doublequant.py:103-113).  Exact in fp64: within a binade the grid is
// uniform, so round-half-up of the scaled mantissa is the midpoint rule.
__device__ __forceinline__ double pow2_d(int k) {  // 2^k for normal exponents, exact
  return __longlong_as_double((long long)((unsigned long long)(1023 + k) << 52));
}
__device__ __forceinline__ unsigned fp8_encode(double q, int E, int M, int B, double maxv) {
  // nearest grid value, ties away from zero (doublequant.py:103-113): within a
  // binade the grid is uniform, so it is round-half-up of the exactly scaled
  // magnitude; the power-of-two scalings and the frexp split act on the bits
  const double a = fabs(q);
  unsigned mag;
  // round half up without the fp64 add (floor(t + 0.5) rounds 0.5 - 2^-54 up)
  auto rhu = [](double t) -> unsigned {
    const double n = floor(t);
    return (unsigned)n + (t - n >= 0.5 ? 1u : 0u);  // t - n is exact
  };
  if (a >= maxv) {
    mag = 0x7Fu;
  } else if (a < pow2_d(1 - B)) {
    mag = rhu(a * pow2_d(B + M - 1));                              // subnormal grid step, exact scaling
  } else {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(a);
    const int ex = (int)((bits >> 52) & 0x7FFu) - 1022;           // a = f 2^ex, f in [0.5, 1)
    const double frac = (double)(bits & 0xFFFFFFFFFFFFFull);       // (2f - 1) 2^52, exact
    mag = ((unsigned)(ex - 1 + B) << M) + rhu(frac * pow2_d(M - 52));  // (2f - 1) 2^M, exact
  }
  (void)E;
  if (mag == 0u) return 0u;
  return (q < 0.0 ? 0x80u : 0u) | mag;
}

// exact decode by assembling the fp64 bit pattern (no ldexp)
__device__ __forceinline__ double fp8_decode_fast(unsigned b, const qlrt_fp8spec& sp) {
  const unsigned M = sp.mant_bits;
  const unsigned e = (b >> M) & ((1u << sp.exp_bits) - 1u);
  const unsigned m = b & ((1u << M) - 1u);
  double mag;
  if (e == 0) {  // m * 2^(1-B-M): exact product with a power of two
    mag = (double)m * __longlong_as_double((long long)((unsigned long long)(1023 + 1 - sp.bias - (int)M) << 52));
  } else {
    mag = __longlong_as_double((long long)(((unsigned long long)(e - sp.bias + 1023) << 52) |
                                           ((unsigned long long)m << (52 - M))));
  }
  return (b >> 7) ? -mag : mag;
}

// reconstruct one first-level constant (doublequant.py:190-195): two
// separate fp64 roundings (no FMA contraction), clamp at 0, round to f32.
__device__ __forceinline__ float dq_constant(unsigned code, float c1, float mu,
                                             const qlrt_fp8spec& sp) {
  double d = fp8_decode_fast(code, sp);
  double r = __dadd_rn(__dmul_rn(d, (double)c1), (double)mu);
  r = r > 0.0 ? r : 0.0;
  return __double2float_rn(r);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

}  // namespace qlrt
