// tcgen05 / TMEM / TMA GEMM engine for sm_100a with an in-kernel NF4
// double-dequant producer -- the frozen 4-bit linear of QLoRA
// (reference: QLinear.forward / backward, pkg/src/qlrt/qlora.py:117-167).
//
//   D[M, N] (fp32 in TMEM) = sum_k A[M, k] B[k, N]  (+ an optional second,
//   "augmented" K segment A2 B2 -- the LoRA term folded into the same
//   accumulator: Y^T = W^T X^T + l2^T (sT)^T, dX^T = W dY^T + l1 dT^T).
//
// One CTA per SM, persistent over 128 x BN output tiles.  Warp roles:
//   warp 0      TMA producer (B tiles; A tiles when A is a bf16 tensor)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5   epilogue: tcgen05.ld -> registers -> global (fp32/bf16,
//               row-major or transposed), double-buffered TMEM accumulators
//   warps 6-13  (NF4 only) dequant producer: packed codes + DQ constants from
//               global -> per-block 16-entry bf16 table -> prmt lookups ->
//               128B-swizzled UMMA tile in shared memory
// The W tile is always the A operand (M = 128 W rows/cols), so each
// dequantized weight feeds BN = 256 token columns of MMA.
#include <cstdlib>

#include "qlrt_common.cuh"
#include <mutex>
#include "sm100_ptx.cuh"

namespace qlrt {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;              // one 128B swizzle row of bf16
constexpr int A_STAGE = BM * BK * 2;  // 16 KB
#ifndef QLRT_EPI_WARPS
#define QLRT_EPI_WARPS 4
#endif
// epilogue warps: 4 or 8 (two per TMEM lane quarter, alternate 32-column chunks)
constexpr int kTmaWarp = 0, kMmaWarp = 1, kEpiWarp0 = 2, kNumEpiWarps = QLRT_EPI_WARPS;
constexpr int kXfWarp0 = kEpiWarp0 + kNumEpiWarps;
constexpr int kNumXfWarps = 8;
constexpr int kCstWarp = kXfWarp0 + kNumXfWarps;  // NF4: codes (TMA) + block-constant producer
constexpr int kNF4Threads = (kCstWarp + 1) * 32;  // 480 (4 epilogue warps) or 608 (8)
constexpr int kPlainThreads = (2 + kNumEpiWarps) * 32;

struct Args {
  int M, N;             // output extent (UMMA M rows, N cols)
  int k_iters;          // main segment K / 64
  int k_iters_aug;      // augmented segment K / 64 (0 = none)
  int splits;           // split-K over the main segment (>1 -> fp32 partials)
  int a_mn, b_mn;       // main segment operand majorness (A ignored for NF4)
  int a2_mn, b2_mn;     // augmented segment majorness
  // NF4 A source (nf4_mode 1: A = W^T (fwd), 2: A = W (bwd))
  int nf4_mode;
  const uint8_t* codes;
  const uint8_t* dq_codes;
  const float* c1;
  const float* mu;
  const float* absmax;  // plain constants if dq_codes == nullptr
  const float* consts;  // fp32 block constants [w_rows][kpitch] (prepass; TMA-fed)
  int64_t kpitch;
  int64_t w_rows, w_cols;
  int bs2;
  int bs2_shift;        // log2(bs2) when bs2 is a power of two, else -1
  qlrt_fp8spec spec;
  double values[16];
  // output
  void* out;
  int64_t ldo;
  int out_f32, out_t;
  float alpha;
  float* ws;            // split-K partials [splits][M][N]
  int to_ws;            // force fp32 partials to ws (finished by the reduce kernel)
  int out_split;        // bf16 out: also store lo = bf16(v - hi) at column offset out_split
  int fold;             // reduce: out[:, n] = D[:, n] + D[:, n + fold] for n < fold
  int pair;             // 2-CTA (cta_group::2) 256 x BN tiles
  // stream-K: the (tile, k-iteration) space is cut into equal contiguous ranges,
  // one per unit (CTA or pair); a tile split across units is finished by the
  // unit holding its k = 0 segment (the "owner"), which adds the fp32
  // partials of the later units in unit order (deterministic)
  int streamk;
  float* sk_ws;         // [gridDim.x][BM][BN] fp32 partials (one per CTA)
  int* sk_flags;        // [gridDim.x]; 0 between launches (owners re-arm what they consume), 1 = partial ready
  // cluster split-K (plain GEMMs): a cluster of csplit CTAs shares one tile,
  // CTA rank z owns k-split z; ranks > 0 stage their fp32 partial in their own
  // shared memory and rank 0 sums them over DSMEM in rank order -- no
  // workspace round trip, no reduce launch
  int csplit;
  // NF4, 1-SM MMAs: a 2-CTA cluster works on the same W rows and two adjacent
  // token tiles; each CTA decodes half of every A stage into both CTAs' shared
  // memory (DSMEM stores), halving the per-SM dequant work
  int share;
  // 512-wide pair tiles: work items >= tail_from are half tiles (one N = 256
  // UMMA each) -- the last partial wave of whole tiles is split in two so it
  // finishes in about half the time; 0 = no half tiles
  int tail_from;
  int tma_out;          // D^T bf16 via TMA stores from the epilogue staging tile
  int stagger;          // 512-wide tiles: per-half accumulator release (drain overlaps MMAs)
  int pdl_trigger;      // let the next (PDL) launch be scheduled right after this grid's prologue
  // the augmented B2 operand is the output of the PDL predecessor (an adapter
  // product running beside this grid): no grid-wide wait at the start; the
  // TMA producer waits (griddepcontrol.wait) only before its first augmented load
  int aug_pdl;
  int trigger_dep;      // aug_pdl grid that still lets its PDL dependent launch after the prologue
  int wait_at_end;      // (with aug_pdl, no augmented segment) the grid needs nothing from its PDL
                        // predecessor but does not complete before it (keeps stream order for later work)
  int units_cap;        // > 0: at most this many (pair) units (SMs left to the predecessor)
  int aug_wrap;         // > 0: the augmented A2 operand has only aug_wrap K rows/cols and is
                        // re-read for K2 = 2 aug_wrap ([l | l] without materialising the pair)
  int cl2;              // plain 1-SM grid launched as 2-CTA clusters (independent CTAs): it
                        // occupies whole SM pairs beside a pair grid instead of fragmenting them
  // sibling projections concatenated along M (grouped forward): tile rows
  // [g aug_gn, (g + 1) aug_gn) take their augmented B2 segment at K offset
  // g aug_gstride (each member's [Ts_hi | Ts_lo] block of Ts_cat)
  int aug_gn, aug_gstride;
  int64_t aug_b2k;      // > 0: B2's own K extent (the whole Ts_cat row)
  // grouped-K skinny GEMM (the members' dT in one launch): output columns
  // [g kg_n, (g + 1) kg_n) reduce over K range [g kg_k, (g + 1) kg_k) of A and
  // B, and read B rows [0, kg_n); kg_kfull = the operands' whole K extent
  int kg_n;
  int64_t kg_k, kg_kfull;
};

#ifndef QLRT_MERGE_FULL
#define QLRT_MERGE_FULL 1
#endif
#ifndef QLRT_EPI_FRAG
#define QLRT_EPI_FRAG 1  // fragment-layout TMEM loads + stmatrix for the staged D^T epilogue
#endif
#ifndef QLRT_ISSUE_E
#define QLRT_ISSUE_E 2  // MMA issue: 2 = elect.sync region (uniform datapath), 0 = lane-0 issue (old)
#endif

#ifndef SKINNY128_STAGES
#define SKINNY128_STAGES 3
#endif
#ifndef SKINNY_STAGES
#define SKINNY_STAGES 4
#endif
template <int BN, bool NF4, bool PAIR = false>
struct Smem {
  static constexpr int BNC = PAIR ? BN / 2 : BN;       // B rows (tokens) held by this CTA
  static constexpr int B_STAGE = BNC * BK * 2;
  static constexpr int EPI_BYTES = kNumEpiWarps * 32 * 32 * 2;  // 32x32 bf16 transpose tile per warp
  // NF4: a separate, decoupled ring of packed codes (4 KB = 128 x 64 nibbles)
  // plus the fp32 block constants of each A stage
  static constexpr int CODE_BYTES = 4096, CONST_BYTES = 2048;
  static constexpr int CST = NF4 ? (BNC >= 128 ? 4 : 8) : 0;
  static constexpr int CRING = CST * (CODE_BYTES + CONST_BYTES);
  // as many A/B stages as fit in ~226 KB, at most 8, even
  static constexpr int FIT = (226 * 1024 - EPI_BYTES - CRING) / (A_STAGE + B_STAGE);
  // skinny plain GEMMs (BN <= 128, the adapter products): few stages, so two
  // CTAs fit per SM and independent skinny GEMMs can run concurrently
  static constexpr int CAP = (!NF4 && BN <= 64) ? SKINNY_STAGES : ((!NF4 && BN <= 128) ? SKINNY128_STAGES : 8);
  // (the NF4 producers alternate stages between groups: even count there)
  static constexpr int STAGES = NF4 ? ((FIT > CAP ? CAP : FIT) & ~1) : (FIT > CAP ? CAP : FIT);
  static constexpr int C_OFF = STAGES * (A_STAGE + B_STAGE);
  static constexpr int EPI_OFF = C_OFF + CRING;
  static constexpr int BAR_OFF = EPI_OFF + EPI_BYTES;
  // full[S], afull[S], empty[S], cfull[CST], cempty[CST], tmem_full[2], tmem_empty[2], tmem_ptr
  static constexpr int BYTES = BAR_OFF + (3 * STAGES + 2 * CST + 4) * 8 + 16 + 1024;  // + align slack
  static_assert(STAGES >= 2 && BYTES <= 232448, "shared memory budget");
};

__device__ __forceinline__ void tile_coords(int t, int m_tiles, int n_tiles, int& mt, int& nt, int& z) {
  const int per = m_tiles * n_tiles;
  z = t / per;
  const int r = t - z * per;
  mt = r / n_tiles;
  nt = r - mt * n_tiles;
}

constexpr int kSkMaxSplit = 4;

// Walks the segments (tile, [i0, i1)) of one unit: round-robin whole tiles, or
// (stream-K) the unit's contiguous share of tiles x T iterations.
struct Sched {
  long long g, g1, T;
  int t, n_tiles_total, n_units, streamk;
  __device__ Sched(int unit, int n_units_, int n_tiles_total_, int T_, int streamk_)
      : T(T_), t(unit), n_tiles_total(n_tiles_total_), n_units(n_units_), streamk(streamk_) {
    const long long G = (long long)n_tiles_total_ * T_;
    g = G * unit / n_units_;
    g1 = G * (unit + 1) / n_units_;
  }
  // full-tile mode: i1 = T (the caller clips split-K tiles to their own extent)
  __device__ bool next(int& tile, int& i0, int& i1) {
    if (!streamk) {
      if (t >= n_tiles_total) return false;
      tile = t;
      i0 = 0;
      i1 = (int)T;
      t += n_units;
      return true;
    }
    if (g >= g1) return false;
    tile = (int)(g / T);
    i0 = (int)(g - (long long)tile * T);
    const long long e = (long long)tile * T + T < g1 ? (long long)tile * T + T : g1;
    i1 = (int)(e - (long long)tile * T);
    g = e;
    return true;
  }
  // first unit whose range starts at or after global iteration x
  __device__ static long long range_begin(long long G, int unit, int n_units_) { return G * unit / n_units_; }
};

// exact decode of the DQ 8-bit float by assembling the fp64 bit pattern
__device__ __forceinline__ double fp8_decode_bits(unsigned b, const qlrt_fp8spec& sp, double sub_scale) {
  const unsigned M = sp.mant_bits;
  const unsigned e = (b >> M) & ((1u << sp.exp_bits) - 1u);
  const unsigned m = b & ((1u << M) - 1u);
  double mag;
  if (e == 0) {
    mag = (double)m * sub_scale;  // m * 2^(1-B-M), exact
  } else {
    const unsigned long long bits = ((unsigned long long)(e - sp.bias + 1023) << 52) |
                                    ((unsigned long long)m << (52 - M));
    mag = __longlong_as_double((long long)bits);
  }
  return (b >> 7) ? -mag : mag;
}

// ---------------------------------------------------------------------------
// NF4 -> bf16 tile producer helpers
// ---------------------------------------------------------------------------
// 16-entry table bf16(v_i * c) (fp32 product) split into lo/hi byte planes (4 regs each)
__device__ __forceinline__ void build_planes(const float (&v)[16], float c, uint32_t (&L)[4], uint32_t (&H)[4]) {
  uint32_t P[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) P[j] = pack_bf16x2(v[2 * j] * c, v[2 * j + 1] * c);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    L[q] = ptx::prmt(P[2 * q], P[2 * q + 1], 0x6420);
    H[q] = ptx::prmt(P[2 * q], P[2 * q + 1], 0x7531);
  }
}

// 8 codes (the nibbles of w, element order) -> 8 bf16 packed in 4 words.
// Selector bookkeeping runs on the FMA pipe (mul.hi for the right shifts) so
// the ALU pipe -- the co-limiter of the fused GEMM -- sees 2 LOP3 + 16 PRMT.
__device__ __forceinline__ void lookup8(uint32_t w, const uint32_t (&L)[4], const uint32_t (&H)[4], uint32_t k3210,
                                        uint32_t& o0, uint32_t& o1, uint32_t& o2, uint32_t& o3) {
  const uint32_t sel = w & 0x77777777u;
  const uint32_t bs = (__umulhi(w, 0x80000000u) & 0x44444444u) | k3210;  // bit 3 of each code -> byte select
  const uint32_t selh = __umulhi(sel, 0x10000u), bsh = __umulhi(bs, 0x10000u);
  const uint32_t la = ptx::prmt(ptx::prmt(L[0], L[1], sel), ptx::prmt(L[2], L[3], sel), bs);
  const uint32_t ha = ptx::prmt(ptx::prmt(H[0], H[1], sel), ptx::prmt(H[2], H[3], sel), bs);
  const uint32_t lb = ptx::prmt(ptx::prmt(L[0], L[1], selh), ptx::prmt(L[2], L[3], selh), bsh);
  const uint32_t hb = ptx::prmt(ptx::prmt(H[0], H[1], selh), ptx::prmt(H[2], H[3], selh), bsh);
  o0 = ptx::prmt(la, ha, 0x5140);
  o1 = ptx::prmt(la, ha, 0x7362);
  o2 = ptx::prmt(lb, hb, 0x5140);
  o3 = ptx::prmt(lb, hb, 0x7362);
}

// one accumulator row segment of EC fp32 values -> global
template <int EC>
__device__ __forceinline__ void store_chunk(const Args& p, const uint32_t (&r)[EC], int64_t m, int64_t n0, int z) {
  const bool full_chunk = n0 + EC <= p.N;
  if ((p.splits > 1 && !p.csplit) || p.to_ws) {
    float* dst = p.ws + ((int64_t)z * p.M + m) * p.N + n0;
    if (full_chunk && (p.N & 3) == 0) {
#pragma unroll
      for (int j = 0; j < EC; j += 4)
        *reinterpret_cast<float4*>(dst + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                          __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
    } else {
#pragma unroll
      for (int j = 0; j < EC; ++j)  // (unrolled + predicated: r stays in registers)
        if (n0 + j < p.N) dst[j] = __uint_as_float(r[j]);
    }
    return;
  }
  // direct output: with fold the logical width is fold (columns n and n + fold summed by the caller)
  const int64_t NL = p.fold ? p.fold : p.N;
  const bool full_out = n0 + EC <= NL;
  const float a = p.alpha;
  if (p.out_t) {  // D^T: out[n][m]; lanes are consecutive m -> coalesced per column
    if (p.out_f32) {
      float* o = static_cast<float*>(p.out);
#pragma unroll
      for (int j = 0; j < EC; ++j)
        if (n0 + j < NL) o[(n0 + j) * p.ldo + m] = __uint_as_float(r[j]) * a;
    } else {
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out);
#pragma unroll
      for (int j = 0; j < EC; ++j)
        if (n0 + j < NL) o[(n0 + j) * p.ldo + m] = __float2bfloat16_rn(__uint_as_float(r[j]) * a);
    }
    return;
  }
  if (p.out_f32) {
    float* o = static_cast<float*>(p.out) + m * p.ldo + n0;
    if (full_out && (p.ldo & 3) == 0) {
#pragma unroll
      for (int j = 0; j < EC; j += 4)
        *reinterpret_cast<float4*>(o + j) = make_float4(__uint_as_float(r[j]) * a, __uint_as_float(r[j + 1]) * a,
                                                        __uint_as_float(r[j + 2]) * a, __uint_as_float(r[j + 3]) * a);
    } else {
#pragma unroll
      for (int j = 0; j < EC; ++j)
        if (n0 + j < NL) o[j] = __uint_as_float(r[j]) * a;
    }
  } else if (p.out_split) {  // bf16 hi/lo pair: v ~= hi + lo to ~16 mantissa bits
    // column n of a member of width out_split -> [hi | lo] block of that member
    // (n0 % out_split + EC <= out_split: a chunk stays inside one member)
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + m * p.ldo + n0 + (n0 / p.out_split) * p.out_split;
#pragma unroll
    for (int j = 0; j < EC; ++j) {
      if (n0 + j >= NL) continue;
      const float v = __uint_as_float(r[j]) * a;
      const __nv_bfloat16 hi = __float2bfloat16_rn(v);
      o[j] = hi;
      o[j + p.out_split] = __float2bfloat16_rn(v - __bfloat162float(hi));
    }
  } else {
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + m * p.ldo + n0;
    if (full_out && (p.ldo & 7) == 0) {
#pragma unroll
      for (int j = 0; j < EC; j += 8)
        *reinterpret_cast<uint4*>(o + j) =
            make_uint4(pack_bf16x2(__uint_as_float(r[j]) * a, __uint_as_float(r[j + 1]) * a),
                       pack_bf16x2(__uint_as_float(r[j + 2]) * a, __uint_as_float(r[j + 3]) * a),
                       pack_bf16x2(__uint_as_float(r[j + 4]) * a, __uint_as_float(r[j + 5]) * a),
                       pack_bf16x2(__uint_as_float(r[j + 6]) * a, __uint_as_float(r[j + 7]) * a));
    } else {
#pragma unroll
      for (int j = 0; j < EC; ++j)
        if (n0 + j < NL) o[j] = __float2bfloat16_rn(__uint_as_float(r[j]) * a);
    }
  }
}

// ---------------------------------------------------------------------------
// the kernel
// PAIR: a 2-CTA cluster computes a 256 x BN tile with tcgen05.mma.cta_group::2;
// each CTA owns 128 rows of A (its half of M, dequantized or TMA-loaded into
// its own smem) and BN/2 rows of B; the leader (rank 0) issues the MMAs, the
// byte counts and producer arrivals of both CTAs land on the leader's
// barriers, and its commits are multicast to both CTAs.
// ---------------------------------------------------------------------------
// QLRT_TRACE builds (tools/trace_gemm.py): per-CTA clock64 totals of where
// each warp role waits, read back with qlrt_trace_fetch.  Not in the product build.
#ifdef QLRT_TRACE
constexpr int kTrSlots = 24;
__device__ unsigned long long g_trace[2 * kNumSMs][kTrSlots];
#define TRW(acc, stmt)                      \
  {                                         \
    const long long _t0 = clock64();        \
    stmt;                                   \
    acc += (unsigned long long)(clock64() - _t0); \
  }
#define TRDECL(...) unsigned long long __VA_ARGS__
#define TRPUT(slot, v) atomicAdd(&g_trace[blockIdx.x % (2 * kNumSMs)][slot], (unsigned long long)(v))
#else
#define TRW(acc, stmt) stmt
#define TRDECL(...)
#define TRPUT(slot, v)
#endif

template <int BN, bool NF4, bool PAIR>
__global__ void __launch_bounds__(NF4 ? kNF4Threads : kPlainThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmO,
                const __grid_constant__ Args p) {
  using L = Smem<BN, NF4, PAIR>;
  constexpr int STAGES = L::STAGES;
  constexpr int CST = L::CST > 0 ? L::CST : 1;
  constexpr int BMP = PAIR ? 2 * BM : BM;   // M rows per (pair) tile
  constexpr int BNC = L::BNC;               // B rows per CTA
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint8_t* sC = smem + L::C_OFF;                       // NF4 codes ring: [CST][4 KB]
  float* sK = reinterpret_cast<float*>(smem + L::C_OFF + L::CST * L::CODE_BYTES);  // constants ring
  __nv_bfloat16* sE = reinterpret_cast<__nv_bfloat16*>(smem + L::EPI_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* full = bars;
  // NF4 (QLRT_MERGE_FULL): the dequant warps arrive on full[] itself, so the
  // MMA issuer waits on one barrier per stage (B bytes + decoded A)
  uint64_t* afull = QLRT_MERGE_FULL ? bars : bars + STAGES;
  uint64_t* empty = bars + 2 * STAGES;
  uint64_t* cfull = bars + 3 * STAGES;
  uint64_t* cempty = cfull + L::CST;
  uint64_t* tfull = cempty + L::CST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* pready = tempty + 3;  // cluster split-K: peers' partials staged (rank 0)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? ptx::cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const bool csplit = !NF4 && !PAIR && p.csplit > 1;
  const bool share = NF4 && !PAIR && p.share;
  const uint32_t srank = share ? ptx::cluster_ctarank() : 0u;  // token-tile half of the shared-decode pair
  const uint32_t zrank = csplit ? ptx::cluster_ctarank() : 0u;  // k-split of this CTA (cluster split-K)
  // work unit = one (pair) tile; a cluster walks the tile list.  Cluster
  // split-K: one (tile, split) per CTA, t = z * tiles + tile
  int unit0 = (PAIR || share) ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  int n_units = (PAIR || share) ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  // accumulators: double-buffered up to BN = 256; BN = 512 (pair tiles of
  // 256 x 512, two N = 256 UMMAs per k-step) fills TMEM with one buffer
  constexpr int NACC = 2 * BN <= 512 ? 2 : 1;
  constexpr uint32_t kNTmemCols = NACC * BN < 32 ? 32 : NACC * BN;
  constexpr int UN = BN > 256 ? 256 : BN;   // N of one UMMA
  constexpr int NUM = BN / UN;              // UMMAs per k16 step
  static_assert(!(BN > 256) || PAIR, "BN = 512 needs 2-CTA pairs");
  const int m_tiles = (p.M + BMP - 1) / BMP;
  const int n_tiles_real = (p.N + BN - 1) / BN;
  const int n_tiles = share ? (n_tiles_real + 1) / 2 : n_tiles_real;  // scheduling grid (pairs of token tiles)
  const int n_tiles_total0 = m_tiles * n_tiles * p.splits;
  const bool halves = NUM > 1 && p.tail_from > 0 && p.tail_from < n_tiles_total0;
  // work items: whole tiles [0, tail_from), then two half tiles per remaining tile
  const int n_tiles_total = halves ? p.tail_from + 2 * (n_tiles_total0 - p.tail_from) : n_tiles_total0;
  const int kc = (p.k_iters + p.splits - 1) / p.splits;
  if (csplit) {
    unit0 = (int)zrank * (m_tiles * n_tiles) + (int)(blockIdx.x / p.csplit);
    n_units = n_tiles_total;  // exactly one segment per CTA
  }
  // iterations of a whole tile (stream-K needs splits == 1)
  const int T_tile = p.streamk ? p.k_iters + p.k_iters_aug : (1 << 30);
  // item -> tile and half (-1 = whole tile; 0 / 1 = which N = 256 half)
  auto item_half = [&](int item, int& tile) -> int {
    if (!halves || item < p.tail_from) { tile = item; return -1; }
    tile = p.tail_from + (item - p.tail_from) / 2;
    return (item - p.tail_from) & 1;
  };
  auto seg_extent = [&](int item, int& mt, int& nt, int& z, int& kb, int& nk, int& total) {
    int tile;
    item_half(item, tile);
    tile_coords(tile, m_tiles, n_tiles, mt, nt, z);
    if (share) nt = 2 * nt + (int)srank;
    kb = z * kc;
    nk = min(kc, p.k_iters - kb);
    total = nk + (p.splits == 1 ? p.k_iters_aug : 0);
  };

  if (warp == kTmaWarp && lane == 0) {
    ptx::prefetch_tmap(&tmB);
    if (!NF4) ptx::prefetch_tmap(&tmA);
    if (NF4) { ptx::prefetch_tmap(&tmC); ptx::prefetch_tmap(&tmK); }
    if (p.k_iters_aug) { ptx::prefetch_tmap(&tmA2); ptx::prefetch_tmap(&tmB2); }
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1 + ((NF4 && QLRT_MERGE_FULL) ? (PAIR ? 8 : 4) : 0));
      // one elected lane per dequant warp (share: this CTA's 2 + the peer's 2)
      if (!QLRT_MERGE_FULL) ptx::mbar_init(&afull[s], NF4 ? (PAIR ? 8 : 4) : 1);
      ptx::mbar_init(&empty[s], share ? 2 : 1);  // share: both CTAs' MMAs read the stage
    }
    for (int c = 0; c < L::CST; ++c) {
      ptx::mbar_init(&cfull[c], 1);      // TMA expect_tx arrival (codes + constants bytes)
      ptx::mbar_init(&cempty[c], share ? 2 : 4);  // one elected lane per warp of the consuming dequant group
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], (PAIR ? 2 : 1) * kNumEpiWarps);  // one lane per epilogue warp
    }
    if (csplit) ptx::mbar_init(pready, (uint32_t)(p.csplit - 1) * kNumEpiWarps);
    ptx::fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    if (PAIR) ptx::tmem_alloc_pair(tmem_slot, kNTmemCols);
    else ptx::tmem_alloc(tmem_slot, kNTmemCols);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (PAIR || csplit || share) ptx::cluster_sync();  // peer barriers initialised before any remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic dependent launch: the prologue above (barriers, TMEM,
  // descriptor prefetch) overlaps the previous kernel's tail; no global data
  // of the previous kernel is touched before this point
  if (!p.aug_pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  // the dependent launch (a split-K reduce, the next GEMM) may be scheduled
  // now: its prologue / launch latency overlaps this grid; it still waits for
  // our completion (griddepcontrol.wait) before touching our outputs
  if (p.pdl_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // leader-side barrier addresses (shared::cluster) for remote arrivals / TMA bytes
  auto leader_addr = [&](uint64_t* bar) -> uint32_t {
    return PAIR ? ptx::mapa_shared(ptx::smem_u32(bar), 0) : ptx::smem_u32(bar);
  };
  auto arrive_leader = [&](uint64_t* bar) {
    if (PAIR) ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(bar), 0));
    else ptx::mbar_arrive(bar);
  };
  auto wait_x = [&](uint64_t* bar, uint32_t ph) {
    if (PAIR) ptx::mbar_wait_cluster(bar, ph);
    else ptx::mbar_wait(bar, ph);
  };
  auto tma = [&](const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1) {
    if (PAIR) ptx::tma_load_2d_pair(m, leader_addr(bar), dst, c0, c1);
    else ptx::tma_load_2d(m, bar, dst, c0, c1);
  };

  if (warp == kTmaWarp) {
    // ======================= TMA producer (every CTA loads its own halves) =======================
    if (lane == 0) {
      uint32_t it = 0;
      bool aug_ready = false;
      TRDECL(tr_we = 0);
      Sched sc(unit0, n_units, n_tiles_total, T_tile, p.streamk);
      int tile, i0, i1;
      while (sc.next(tile, i0, i1)) {
        int mt, nt, z, kb, nk, total;
        seg_extent(tile, mt, nt, z, kb, nk, total);
        i1 = min(i1, total);
        const int m_cta = mt * BMP + (int)rank * BM;
        const int n_cta = nt * BN + (int)rank * BNC;
        for (int i = i0; i < i1; ++i, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          TRW(tr_we, ptx::mbar_wait(&empty[s], ph ^ 1));
          const bool aug = i >= nk;
          const CUtensorMap* ma = aug ? &tmA2 : &tmA;
          const CUtensorMap* mb = aug ? &tmB2 : &tmB;
          const int amn = aug ? p.a2_mn : p.a_mn;
          const int bmn = aug ? p.b2_mn : p.b_mn;
          const int k0 = (aug ? (i - nk) : (kb + i)) * BK;
          // wrap: A2 holds aug_wrap K lines per group of 2 aug_wrap (hi and lo of
          // each member's pair multiply the same l rows / columns)
          const int k0a = (aug && p.aug_wrap) ? (k0 / (2 * p.aug_wrap)) * p.aug_wrap + k0 % p.aug_wrap : k0;
          const int k0b = (aug && p.aug_gn) ? k0 + ((mt * BMP) / p.aug_gn) * p.aug_gstride : k0;
          const int kgg = (!aug && p.kg_n) ? (nt * BN) / p.kg_n : 0;  // grouped-K member of this column tile
          const int kadd = kgg * (int)p.kg_k, nsub = kgg * p.kg_n;
          const bool a_tma = aug || !NF4;
          if (aug && p.aug_pdl && !aug_ready) {  // B2 = the adapter product of the PDL predecessor
            asm volatile("griddepcontrol.wait;" ::: "memory");
            aug_ready = true;
          }
          int tdummy;
          const int hh = item_half(tile, tdummy);
          const int b_bytes = hh >= 0 ? L::B_STAGE / NUM : L::B_STAGE;
          if (leader)  // one arrival per phase; both CTAs' bytes
            ptx::mbar_arrive_expect_tx(&full[s], (PAIR ? 2 : 1) * (b_bytes + (a_tma ? A_STAGE : 0)));
          uint8_t* a_dst = sA + s * A_STAGE;
          uint8_t* b_dst = sB + s * L::B_STAGE;
          if (a_tma) {
            if (amn) {
              tma(ma, &full[s], a_dst, m_cta, k0a + kadd);
              tma(ma, &full[s], a_dst + 8192, m_cta + 64, k0a + kadd);
            } else {
              tma(ma, &full[s], a_dst, k0a + kadd, m_cta);
            }
          }
          if (bmn) {
#pragma unroll
            for (int j = 0; j < (BNC + 63) / 64; ++j) tma(mb, &full[s], b_dst + j * 8192, n_cta + j * 64, k0b);
          } else if (NUM > 1) {  // one 128-token half of each UMMA's B, at the same offset in both CTAs
#pragma unroll
            for (int j = 0; j < NUM; ++j)
              if (hh < 0 || hh == j)
                tma(mb, &full[s], b_dst + j * (L::B_STAGE / NUM), k0b, nt * BN + j * UN + (int)rank * (UN / 2));
          } else {
            tma(mb, &full[s], b_dst, k0b + kadd, n_cta - nsub);
          }
        }
      }
      TRPUT(9, tr_we);
    }
  } else if (warp == kMmaWarp) {
    // ======================= MMA issuer (leader only) =======================
    if (leader) {
      uint32_t it = 0, local = 0;
      TRDECL(tr_wt = 0, tr_wf = 0, tr_wa = 0, tr_is = 0);
      TRDECL(tr_t0 = clock64());
      Sched sc(unit0, n_units, n_tiles_total, T_tile, p.streamk);
      int tile, i0, i1;
      for (; sc.next(tile, i0, i1); ++local) {
        int mt, nt, z, kb, nk, total;
        seg_extent(tile, mt, nt, z, kb, nk, total);
        i1 = min(i1, total);
        const uint32_t acc = local % NACC;
        int tdummy;
        const int hh = item_half(tile, tdummy);
        // 512-wide tiles (one accumulator): the epilogue frees the two 256-column
        // halves separately (tempty[0], tempty[1]); the first `pre` stages of
        // the tile issue their half-0 MMAs as soon as half 0 is drained and
        // their half-1 MMAs once half 1 is, so the drain overlaps the MMAs
        const bool split = NUM == 2 && NACC == 1 && p.stagger;
        const int pre = (split && hh < 0) ? min(STAGES, i1 - i0) : 0;
        if (split) {
          wait_x(&tempty[0], (local & 1) ^ 1);
          if (pre == 0) wait_x(&tempty[1], (local & 1) ^ 1);
        } else {
          TRW(tr_wt, wait_x(&tempty[acc], ((local / NACC) & 1) ^ 1));
        }
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        auto issue = [&](int i, int s, int jsel, bool commit) {  // jsel: -1 both halves, else that half
          const bool aug = i >= nk;
          const int amn = aug ? p.a2_mn : (NF4 ? (p.nf4_mode == 1) : p.a_mn);
          const int bmn = aug ? p.b2_mn : p.b_mn;
          const uint32_t idesc = ptx::idesc_bf16(BMP, UN, amn, bmn);
          const uint32_t a_addr = ptx::smem_u32(sA + s * A_STAGE);
          const uint32_t b_addr = ptx::smem_u32(sB + s * L::B_STAGE);
#if QLRT_ISSUE_E == 2
          // one elected thread (elect.sync: ptxas keeps the region on the
          // uniform datapath); descriptors built once per stage, then + 2048 B
          // (MN-major) or + 32 B (K-major) per k16 step in the >> 4 address field
          if (ptx::elect_one()) {
            const uint32_t idesc2 = ptx::idesc_bf16(BMP, UN, amn, bmn);
            const uint64_t ad0 = amn ? ptx::sdesc_sw128(a_addr, 8192, 1024) : ptx::sdesc_sw128(a_addr, 16, 1024);
            const uint64_t astep = amn ? 128u : 2u, bstep = bmn ? 128u : 2u;
            uint64_t bd0[NUM];
#pragma unroll
            for (int j = 0; j < NUM; ++j) {
              const uint32_t bj = b_addr + (uint32_t)(j * (L::B_STAGE / NUM));
              bd0[j] = bmn ? ptx::sdesc_sw128(bj, 8192, 1024) : ptx::sdesc_sw128(bj, 16, 1024);
            }
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
#pragma unroll
              for (int j = 0; j < NUM; ++j) {
                if ((hh >= 0 && hh != j) || (jsel >= 0 && jsel != j)) continue;
                const uint64_t ad = ad0 + kk * astep, bd = bd0[j] + kk * bstep;
                if (PAIR) ptx::umma_bf16_pair(d_tmem + j * UN, ad, bd, idesc2, (i != i0) || kk != 0);
                else ptx::umma_bf16(d_tmem + j * UN, ad, bd, idesc2, (i != i0) || kk != 0);
              }
            }
            if (commit) {
              if (PAIR) ptx::umma_commit_pair_mc(&empty[s], 0x3);
              else if (share) ptx::umma_commit_mc(&empty[s], 0x3);
              else ptx::umma_commit(&empty[s]);
            }
          }
#else
          if (lane == 0) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ad = amn ? ptx::sdesc_sw128(a_addr + kk * 2048, 8192, 1024)
                                      : ptx::sdesc_sw128(a_addr + kk * 32, 16, 1024);
#pragma unroll
              for (int j = 0; j < NUM; ++j) {
                if ((hh >= 0 && hh != j) || (jsel >= 0 && jsel != j)) continue;
                const uint32_t bj = b_addr + (uint32_t)(j * (L::B_STAGE / NUM));
                const uint64_t bd = bmn ? ptx::sdesc_sw128(bj + kk * 2048, 8192, 1024)
                                        : ptx::sdesc_sw128(bj + kk * 32, 16, 1024);
                if (PAIR) ptx::umma_bf16_pair(d_tmem + j * UN, ad, bd, idesc, (i != i0) || kk != 0);
                else ptx::umma_bf16(d_tmem + j * UN, ad, bd, idesc, (i != i0) || kk != 0);
              }
            }
            if (commit) {
              if (PAIR) ptx::umma_commit_pair_mc(&empty[s], 0x3);
              else if (share) ptx::umma_commit_mc(&empty[s], 0x3);  // frees the slot in both CTAs
              else ptx::umma_commit(&empty[s]);
            }
          }
#endif
          __syncwarp();
        };
        if (pre > 0) {
          for (int q = 0; q < pre; ++q) {  // half 0 of the first stages
            const uint32_t itq = it + (uint32_t)q;
            const int s = itq % STAGES;
            wait_x(&full[s], (itq / STAGES) & 1);
            if (NF4 && !QLRT_MERGE_FULL) wait_x(&afull[s], (itq / STAGES) & 1);
            ptx::tc_fence_after();
            issue(i0 + q, s, 0, false);
          }
          wait_x(&tempty[1], (local & 1) ^ 1);
          ptx::tc_fence_after();
          for (int q = 0; q < pre; ++q, ++it) issue(i0 + q, it % STAGES, 1, true);  // their half 1
        }
        for (int i = i0 + pre; i < i1; ++i, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          TRW(tr_wf, wait_x(&full[s], ph));
          if (NF4 && !QLRT_MERGE_FULL) TRW(tr_wa, wait_x(&afull[s], ph));
          ptx::tc_fence_after();
          TRW(tr_is, issue(i, s, -1, true));
        }
#if QLRT_ISSUE_E == 2
        if (ptx::elect_one()) {
          if (PAIR) ptx::umma_commit_pair_mc(&tfull[acc], 0x3);
          else ptx::umma_commit(&tfull[acc]);
        }
#else
        if (lane == 0) {
          if (PAIR) ptx::umma_commit_pair_mc(&tfull[acc], 0x3);
          else ptx::umma_commit(&tfull[acc]);
        }
#endif
        __syncwarp();
      }
      if (lane == 0) {
        TRPUT(0, tr_wt); TRPUT(1, tr_wf); TRPUT(2, tr_wa); TRPUT(3, clock64() - tr_t0); TRPUT(11, local); TRPUT(12, tr_is);
      }
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kNumEpiWarps) {
    // ======================= epilogue (each CTA drains its own TMEM rows) =======================
    constexpr int EC = BN < 32 ? BN : 32;   // columns per tcgen05.ld
    const int quarter = warp & 3;           // TMEM lane quarter this warp may access
    const int csub = (warp - kEpiWarp0) >> 2;  // which alternate 32-column chunks (8 epilogue warps)
    constexpr int CSTEP = (kNumEpiWarps / 4) * (BN < 32 ? BN : 32);
    const int row = quarter * 32 + lane;    // accumulator row (M index within this CTA's half)
    uint32_t local = 0;
    TRDECL(tr_wt = 0, tr_dr = 0, tr_d0 = 0);
    Sched sc(unit0, n_units, n_tiles_total, T_tile, p.streamk);
    const long long G = (long long)n_tiles_total * T_tile;
    int tile, i0, i1;
    for (; sc.next(tile, i0, i1); ++local) {
      int mt, nt, z, kb, nk, total;
      seg_extent(tile, mt, nt, z, kb, nk, total);
      i1 = min(i1, total);
      // stream-K: a segment not starting at k = 0 leaves an fp32 partial; the
      // k = 0 segment (owner) adds the partials of units unit0+1 .. v_end-1
      const bool partial = p.streamk && i0 != 0;
      int v_end = unit0 + 1;
      if (p.streamk && i0 == 0 && i1 < total)
        while (v_end < n_units && Sched::range_begin(G, v_end, n_units) < (long long)(tile + 1) * T_tile) ++v_end;
      const uint32_t acc = local % NACC;
      TRW(tr_wt, ptx::mbar_wait(&tfull[acc], (local / NACC) & 1));
#ifdef QLRT_TRACE
      tr_d0 = clock64();
#endif
      ptx::tc_fence_after();
      if (v_end > unit0 + 1) {  // wait for the later units' partials of this tile (one flag per lane)
        for (int v0 = unit0 + 1; v0 < v_end; v0 += 32) {
          const int v = v0 + lane;
          int ready = v < v_end ? 0 : 1;
          const int* f = p.sk_flags + (PAIR ? 2 * v + (int)rank : v);
          while (!__all_sync(0xffffffffu, ready))
            if (!ready) asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(ready) : "l"(f) : "memory");
        }
      }
      const int64_t m_base = (int64_t)mt * BMP + (int64_t)rank * BM;
      const int64_t m = m_base + row;
      // chunk c of the accumulator (+ the stream-K contributors' partials); the
      // partial tile layout per CTA is [column group of 4][row][4]: a warp's
      // float4 accesses cover 512 contiguous bytes
      auto load_acc = [&](int c, uint32_t (&r)[EC]) {
        ptx::tmem_ld<EC>(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + c, r);
        // contributors four at a time, 16 columns at a time: 16 independent L2
        // loads in flight, then the adds in unit order (deterministic)
        for (int v0 = unit0 + 1; v0 < v_end; v0 += 4) {
#pragma unroll
          for (int h = 0; h < EC; h += 16) {
            float4 w[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int v = v0 + q < v_end ? v0 + q : v0;
              const float* src =
                  p.sk_ws + (size_t)(PAIR ? 2 * v + (int)rank : v) * BM * BN + (size_t)c * BM + row * 4;
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) w[q][jj] = __ldcg(reinterpret_cast<const float4*>(src + (h + 4 * jj) * BM));
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (v0 + q >= v_end) break;
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const int j = h + 4 * jj;
                r[j] = __float_as_uint(__uint_as_float(r[j]) + w[q][jj].x);
                r[j + 1] = __float_as_uint(__uint_as_float(r[j + 1]) + w[q][jj].y);
                r[j + 2] = __float_as_uint(__uint_as_float(r[j + 2]) + w[q][jj].z);
                r[j + 3] = __float_as_uint(__uint_as_float(r[j + 3]) + w[q][jj].w);
              }
            }
          }
        }
      };
      // cluster split-K: rank 0 adds ranks 1.. (their smem, [c/4][row][4] fp32) in rank order
      auto add_peers = [&](int c, uint32_t (&r)[EC]) {
        for (int zz = 1; zz < p.csplit; ++zz) {
          const uint32_t base = ptx::mapa_shared(ptx::smem_u32(sA), (uint32_t)zz) + (uint32_t)((c * BM + row * 4) * 4);
#pragma unroll
          for (int j = 0; j < EC; j += 4) {
            float4 w4;
            asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(w4.x), "=f"(w4.y), "=f"(w4.z), "=f"(w4.w)
                         : "r"(base + (uint32_t)(j * BM * 4)));
            r[j] = __float_as_uint(__uint_as_float(r[j]) + w4.x);
            r[j + 1] = __float_as_uint(__uint_as_float(r[j + 1]) + w4.y);
            r[j + 2] = __float_as_uint(__uint_as_float(r[j + 2]) + w4.z);
            r[j + 3] = __float_as_uint(__uint_as_float(r[j + 3]) + w4.w);
          }
        }
      };
      if (csplit && zrank != 0) {  // stage this split's accumulator, signal rank 0, done
        float* st = reinterpret_cast<float*>(sA);
#pragma unroll 1
        for (int c0 = csub * EC; c0 < BN; c0 += CSTEP) {
          uint32_t r[EC];
          ptx::tmem_ld<EC>(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + c0, r);
#pragma unroll
          for (int j = 0; j < EC; j += 4)
            *reinterpret_cast<float4*>(st + (c0 + j) * BM + row * 4) =
                make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                            __uint_as_float(r[j + 3]));
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];"
                       ::"r"(ptx::mapa_shared(ptx::smem_u32(pready), 0)) : "memory");
          arrive_leader(&tempty[acc]);
        }
        continue;
      }
      if (csplit) ptx::mbar_wait_cluster(pready, 0);
      auto store_partial = [&](int c, const uint32_t (&r)[EC]) {
        float* dst = p.sk_ws + (size_t)blockIdx.x * BM * BN + (size_t)c * BM + row * 4;
#pragma unroll
        for (int j = 0; j < EC; j += 4)
          __stcg(reinterpret_cast<float4*>(dst + j * BM), make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                                     __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
      };
      // fold (hi/lo operand pairs, fold <= BN / 2, one column tile): out column
      // n = D[:, n] + D[:, n + fold]
      const bool direct_fold = p.fold && !((p.splits > 1 && !p.csplit) || p.to_ws);  // else the reduce kernel folds
      int tdummy;
      const int hh = item_half(tile, tdummy);
      const int cbeg = hh >= 0 ? hh * UN : 0;  // a half tile drains its own 256 columns
      const int cend = direct_fold ? p.fold : (hh >= 0 ? cbeg + UN : BN);
      // the staged 32 x 32 D^T tile (row j = token n0 + j) out with 16B vector
      // stores: 4 lanes cover one 64B output row segment
      auto store_staged_t = [&](const __nv_bfloat16* st, int64_t n0) {
        const int64_t mcol = m_base + quarter * 32 + (lane & 3) * 8;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int rr = q * 8 + (lane >> 2);
          const int64_t n = n0 + rr;
          const uint4 v = *reinterpret_cast<const uint4*>(st + rr * 32 + (lane & 3) * 8);
          if (n < p.N) {
            __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + n * p.ldo + mcol;
            if (mcol + 8 <= p.M && (p.ldo & 7) == 0) {
              *reinterpret_cast<uint4*>(o) = v;
            } else {
              const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (mcol + u < p.M)
                  reinterpret_cast<unsigned short*>(o)[u] = (unsigned short)(vw[u >> 1] >> (16 * (u & 1)));
            }
          }
        }
        __syncwarp();
      };
      // bf16 D^T through the per-warp staging tile, loaded in the mma fragment
      // layout (tcgen05.ld 16x256b) and transposed by stmatrix: 2 loads + 16
      // packs + 4 stmatrix per 32 x 32 chunk instead of 32 scalar 16-bit stores
      const bool staged_t = EC == 32 && (p.tma_out || (p.out_t && !p.out_f32 && p.splits == 1 && !p.to_ws));
      const bool frag = staged_t && QLRT_EPI_FRAG && !partial && !csplit && v_end == unit0 + 1;
#pragma unroll 1
      for (int c0 = cbeg + csub * EC; c0 < cend && frag; c0 += CSTEP) {
        uint32_t r[32];
        const uint32_t tq = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + c0;
        ptx::tmem_ld_frag32(tq, tq + (16u << 16), r);
        if (direct_fold) {
          uint32_t r2[32];
          ptx::tmem_ld_frag32(tq + p.fold, tq + (16u << 16) + p.fold, r2);
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(r2[j]));
        }
        if (p.alpha != 1.0f) {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * p.alpha);
        }
        const int64_t n0 = (int64_t)nt * BN + c0;
        __nv_bfloat16* st = sE + (warp - kEpiWarp0) * 32 * 32;
        if (p.tma_out && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        // matrix i of each stmatrix = features 8i..8i+7 x tokens 8x..8x+7; this
        // lane addresses stored row (token) 8x + lane % 8 of matrix lane / 8
        const uint32_t sa = ptx::smem_u32(st) + (uint32_t)(((lane & 7) * 32 + 8 * (lane >> 3)) * 2);
#pragma unroll
        for (int x = 0; x < 4; ++x)
          ptx::stmatrix_x4_trans(
              sa + x * 8 * 32 * 2,
              ptx::pack_bf16x2(__uint_as_float(r[4 * x]), __uint_as_float(r[4 * x + 1])),
              ptx::pack_bf16x2(__uint_as_float(r[4 * x + 2]), __uint_as_float(r[4 * x + 3])),
              ptx::pack_bf16x2(__uint_as_float(r[16 + 4 * x]), __uint_as_float(r[16 + 4 * x + 1])),
              ptx::pack_bf16x2(__uint_as_float(r[16 + 4 * x + 2]), __uint_as_float(r[16 + 4 * x + 3])));
        if (p.tma_out) {
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tmO),
                "r"((int)(m_base + quarter * 32)), "r"((int)n0), "r"(ptx::smem_u32(st))
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else {
          __syncwarp();
          store_staged_t(st, n0);
        }
        if (NUM == 2 && NACC == 1 && p.stagger && hh < 0 && c0 + CSTEP >= UN && c0 < UN) {
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(&tempty[0]);
        }
      }
#pragma unroll 1
      for (int c0 = cbeg + csub * EC; c0 < cend && !frag; c0 += CSTEP) {
        uint32_t r[EC];
        if (partial) {
          ptx::tmem_ld<EC>(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + c0, r);
          store_partial(c0, r);
          if (direct_fold) {
            ptx::tmem_ld<EC>(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + c0 + p.fold, r);
            store_partial(c0 + p.fold, r);
          }
          continue;
        }
        load_acc(c0, r);
        if (csplit) add_peers(c0, r);
        if (direct_fold) {
          uint32_t r2[EC];
          load_acc(c0 + p.fold, r2);
          if (csplit) add_peers(c0 + p.fold, r2);
#pragma unroll
          for (int j = 0; j < EC; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(r2[j]));
        }
        const int64_t n0 = (int64_t)nt * BN + c0;
#ifdef QLRT_HACK_NOEPI
        if (NF4) { if (r[0] == 0x7fffffffu && lane == 99) static_cast<uint32_t*>(p.out)[0] = r[1]; continue; }
#endif
        if (EC == 32 && p.tma_out) {
          // D^T: the 32 x 32 tile staged in shared memory (row = token n0 + j,
          // 32 features), written by one TMA store (clips at the tensor edge);
          // the staging tile is reused once the previous store has read it
          __nv_bfloat16* st = sE + (warp - kEpiWarp0) * 32 * 32;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int j = 0; j < EC; ++j) st[j * 32 + lane] = __float2bfloat16_rn(__uint_as_float(r[j]) * p.alpha);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tmO),
                "r"((int)(m_base + quarter * 32)), "r"((int)n0), "r"(ptx::smem_u32(st))
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else if (EC == 32 && p.out_t && !p.out_f32 && p.splits == 1 && !p.to_ws) {
          // D^T tile through shared memory: row j = token n0+j, 32 features per row,
          // then 16B vector stores (4 lanes cover one 64B output row segment)
          __nv_bfloat16* st = sE + (warp - kEpiWarp0) * 32 * 32;
#pragma unroll
          for (int j = 0; j < EC; ++j) st[j * 32 + lane] = __float2bfloat16_rn(__uint_as_float(r[j]) * p.alpha);
          __syncwarp();
          store_staged_t(st, n0);
        } else if (m < p.M) {
          store_chunk<EC>(p, r, m, n0, z);
        }
        if (NUM == 2 && NACC == 1 && p.stagger && hh < 0 && c0 + CSTEP >= UN && c0 < UN) {
          ptx::tc_fence_before();  // this warp's reads of columns [0, 256) are done
          __syncwarp();
          if (lane == 0) arrive_leader(&tempty[0]);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
#ifdef QLRT_TRACE
      tr_dr += clock64() - tr_d0;
#endif
      if (NUM == 2 && NACC == 1 && p.stagger) {  // half 1 (and half 0 if not released in the loop)
        if (lane == 0) {
          if (!(hh < 0 && !partial)) arrive_leader(&tempty[0]);
          arrive_leader(&tempty[1]);
        }
      } else if (lane == 0) {
        arrive_leader(&tempty[acc]);
      }
      if (v_end > unit0 + 1) {  // every epilogue warp consumed the partials: re-arm the flags
        asm volatile("bar.sync 1, %0;" ::"n"(kNumEpiWarps * 32) : "memory");
        if (warp == kEpiWarp0)
          for (int v = unit0 + 1 + lane; v < v_end; v += 32) p.sk_flags[PAIR ? 2 * v + (int)rank : v] = 0;
      }
      if (partial) {  // all four epilogue warps wrote their rows: publish
        asm volatile("bar.sync 1, %0;" ::"n"(kNumEpiWarps * 32) : "memory");
        if (warp == kEpiWarp0 && lane == 0) {
          __threadfence();
          asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.sk_flags + blockIdx.x), "r"(1) : "memory");
        }
      }
    }
    if (p.tma_out && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (lane == 0 && warp == kEpiWarp0) { TRPUT(4, tr_wt); TRPUT(5, tr_dr); }
  } else if (NF4 && warp == kCstWarp) {
    // ======================= codes + block-constant producer =======================
    // Runs ahead of the dequant warps through its own ring, TMA-loading the
    // packed codes of this CTA's next A half-tile (fwd: W[k0:k0+64, m:m+128]
    // as 64 rows x 64 B; bwd: W[m:m+128, k0:k0+64] as 128 rows x 32 B) and the
    // matching fp32 block constants (fwd: 64 rows x 4; bwd: 128 rows x 4).
    if (lane == 0) {
      uint32_t cit = 0;
      TRDECL(tr_wc = 0);
      const uint32_t kbytes = p.nf4_mode == 1 ? 64 * 16 : 128 * 16;
      Sched sc(unit0, n_units, n_tiles_total, T_tile, p.streamk);
      int tile, i0, i1;
      while (sc.next(tile, i0, i1)) {
        int mt, nt, z, kb, nk, total;
        seg_extent(tile, mt, nt, z, kb, nk, total);
        const int m_cta = mt * BMP + (int)rank * BM;
        for (int i = i0; i < min(i1, nk); ++i, ++cit) {
          const int c = cit % CST;
          const int k0 = (kb + i) * BK;
          TRW(tr_wc, ptx::mbar_wait(&cempty[c], ((cit / CST) & 1) ^ 1));
          ptx::mbar_arrive_expect_tx(&cfull[c], L::CODE_BYTES + kbytes);
          uint8_t* cdst = sC + c * L::CODE_BYTES;
          float* kdst = sK + c * (L::CONST_BYTES / 4);
          if (p.nf4_mode == 1) {
            ptx::tma_load_2d(&tmC, &cfull[c], cdst, m_cta / 2, k0);
            ptx::tma_load_2d(&tmK, &cfull[c], kdst, ((m_cta / 64) & ~3) * 4, k0);  // 16 B aligned start
          } else {
            ptx::tma_load_2d(&tmC, &cfull[c], cdst, k0 / 2, m_cta);
            ptx::tma_load_2d(&tmK, &cfull[c], kdst, ((k0 / 64) & ~3) * 4, m_cta);
          }
        }
      }
      TRPUT(10, tr_wc);
    }
  } else if (NF4 && warp >= kXfWarp0 && warp < kXfWarp0 + kNumXfWarps) {
    // ======================= NF4 dequant producer =======================
    const int xw = warp - kXfWarp0;
    // stages rotate over the groups: 2 groups of 4 warps (128 items each), or
    // with share 4 groups of 2 warps (this CTA's 64 items of every stage)
    const int ngrp = share ? 4 : 2;
    const int grp = share ? xw >> 1 : xw >> 2;
    const int item = share ? (int)srank * 64 + (xw & 1) * 32 + lane  // 0..127: one 64-element W block
                           : (xw & 3) * 32 + lane;
    float vals[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) vals[i] = (float)p.values[i];
    // fwd: item -> (h = item & 1, r = item >> 1): A image at h*8192 + r*128,
    //      codes at r*64 + h*32 (W row k0+r, cols m+64h..+64)
    // bwd: item -> W row m+item, cols k0..k0+64: A image item*128, codes item*32
    // fwd: warp (xw & 3) -> half h = xw & 1 of rows rr = 32 * ((xw & 3) >> 1) + lane: consecutive lanes
    // write consecutive 128 B rows of the MN-major image (conflict-free 16 B stores)
    // share: this CTA decodes column half h = srank, rows rr = 32 * (xw & 1) + lane
    const int h = share ? (int)srank : xw & 1;
    const int rr = share ? 32 * (xw & 1) + lane : 32 * ((xw & 3) >> 1) + lane;
    const bool fwd = p.nf4_mode == 1;
    const uint32_t soff = fwd ? (uint32_t)(h * 8192 + rr * 128) : (uint32_t)(item * 128);
    // the two 16 B halves of an item's 32 code bytes are read in lane-alternating
    // order (fewer bank conflicts); jA = 1 swaps chunk indices 0-3 <-> 4-7
    const uint32_t jA = fwd ? (uint32_t)((rr >> 1) & 1) : (uint32_t)((item >> 2) & 1);
    const uint32_t swz = ((soff >> 7) & 7) ^ (jA << 2);
    const uint32_t codes_s = ptx::smem_u32(sC) + (fwd ? (uint32_t)(rr * 64 + h * 32) : (uint32_t)item * 32);
    // constants tile: fwd [64 rows][4] -> (r, h); bwd [128 rows][4] -> (item, 0)
    const uint32_t consts_s = ptx::smem_u32(sK) + (fwd ? (uint32_t)(rr * 16 + h * 4) : (uint32_t)item * 16);
    const uint32_t k3210 = 0x32103210u;
    const uint32_t a_s = ptx::smem_u32(sA) + soff;
    const uint32_t a_peer = share ? ptx::mapa_shared(a_s, srank ^ 1u) : 0u;  // same offset in the peer CTA
    auto arrive_afull = [&](uint64_t* bar) {  // this CTA's barrier, and (share) the peer's
      arrive_leader(bar);
      if (share) {
#ifdef QLRT_SHARE_RELAXED
        ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(bar), srank ^ 1u));
#else
        ptx::mbar_arrive_cluster_release(ptx::mapa_shared(ptx::smem_u32(bar), srank ^ 1u));
#endif
      }
    };
    uint32_t it = 0, cit = 0;
    TRDECL(tr_wc = 0, tr_we = 0, tr_t0 = clock64());
    Sched sc(unit0, n_units, n_tiles_total, T_tile, p.streamk);
    int tile, i0, i1;
    while (sc.next(tile, i0, i1)) {
      int mt, nt, z, kb, nk, total;
      seg_extent(tile, mt, nt, z, kb, nk, total);
      i1 = min(i1, total);
      const int m_cta = mt * BMP + (int)rank * BM;
      // stages rotate over the groups by the running stage count
      for (int i = i0 + (int)(((uint32_t)grp - it) % (uint32_t)ngrp); i < i1; i += ngrp) {
        const uint32_t my = it + (uint32_t)(i - i0);
        const int s = my % STAGES;
        const uint32_t ph = (my / STAGES) & 1;
        if (i >= nk) {  // augmented (TMA-fed) stage: keep afull's phase in step
          ptx::mbar_wait(&empty[s], ph ^ 1);
          __syncwarp();
          if (lane == 0) arrive_afull(&afull[s]);
          continue;
        }
        const uint32_t ci = cit + (uint32_t)(i - i0);
        const int c = ci % CST;
        // the constants box starts at a 16 B aligned column: index within it
        const uint32_t kcol = (uint32_t)((p.nf4_mode == 1 ? m_cta / 64 : kb + i) & 3) * 4;
        TRW(tr_wc, ptx::mbar_wait(&cfull[c], (ci / CST) & 1));
        const uint4 w0 = ptx::ld_shared_v4(codes_s + c * L::CODE_BYTES + jA * 16);
        const uint4 w1 = ptx::ld_shared_v4(codes_s + c * L::CODE_BYTES + (jA ^ 1u) * 16);
        const float cst = ptx::ld_shared_f32(consts_s + c * L::CONST_BYTES + kcol);
        uint32_t Lp[4], Hp[4];
        build_planes(vals, cst, Lp, Hp);
        TRW(tr_we, ptx::mbar_wait(&empty[s], ph ^ 1));
        const uint32_t base = a_s + s * A_STAGE;
        const uint32_t words[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#ifndef QLRT_HACK_DECODE
#define QLRT_HACK_DECODE 8
#endif
        uint32_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          if (ch < QLRT_HACK_DECODE) lookup8(words[ch], Lp, Hp, k3210, o0, o1, o2, o3);
          ptx::st_shared_v4(base + ((ch ^ swz) << 4), o0, o1, o2, o3);
          if (share) ptx::st_cluster_v4(a_peer + s * A_STAGE + ((ch ^ swz) << 4), o0, o1, o2, o3);
        }
        if (share) ptx::fence_proxy_async_cluster();
        else ptx::fence_proxy_async_smem();
        __syncwarp();  // orders the warp's smem writes before the elected release
        if (lane == 0) {
          arrive_afull(&afull[s]);
          // release the codes slot only now: every loaded word has been consumed
          // (an arrive right after the loads can overtake them, and the next TMA
          // would overwrite the slot under an in-flight ld.shared)
          ptx::mbar_arrive(&cempty[c]);
        }
      }
      it += (uint32_t)(i1 - i0);
      cit += (uint32_t)max(0, min(i1, nk) - i0);
    }
    if (lane == 0) { TRPUT(6, tr_wc); TRPUT(7, tr_we); TRPUT(8, clock64() - tr_t0); }
  }

  ptx::tc_fence_before();
  if (p.wait_at_end) asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  if (PAIR || csplit || share) ptx::cluster_sync();  // (peers stay alive until remote traffic is done)
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    if (PAIR) ptx::tmem_dealloc_pair(tmem_base, kNTmemCols);
    else ptx::tmem_dealloc(tmem_base, kNTmemCols);
  }
}

// split-K reduction: out = alpha * sum_z ws[z]  (fixed order -> deterministic);
// fold > 0 also adds column n + fold into column n (hi/lo operand pairs);
// out_split writes a bf16 hi/lo pair.
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N, int fold, float alpha,
                                     void* __restrict__ out, int64_t ldo, int out_f32, int out_t, int out_split) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (PDL launch: the partials are complete)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t total = (int64_t)M * N;
  const int NO = fold ? N / 2 : N;  // fold: members of 2 fold columns [hi | lo] -> fold columns each
  const int64_t total_o = (int64_t)M * NO;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total_o;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / NO, n = i - m * NO;
    const int64_t src = m * N + (fold ? (n / fold) * 2 * fold + n % fold : n);
    float acc = 0.0f;
    for (int z = 0; z < splits; ++z) {
      acc += ws[(int64_t)z * total + src];
      if (fold) acc += ws[(int64_t)z * total + src + fold];
    }
    acc *= alpha;
    // out_split: column n of a member of width out_split -> its [hi | lo] block
    const int64_t ns = out_split ? n + (n / out_split) * out_split : n;
    const int64_t o = out_t ? ns * ldo + m : m * ldo + ns;
    if (out_f32) {
      static_cast<float*>(out)[o] = acc;
    } else {
      const __nv_bfloat16 hi = __float2bfloat16_rn(acc);
      static_cast<__nv_bfloat16*>(out)[o] = hi;
      if (out_split) static_cast<__nv_bfloat16*>(out)[o + out_split] = __float2bfloat16_rn(acc - __bfloat162float(hi));
    }
  }
}

// double-dequantized block constants of a weight as an fp32 matrix
// [w_rows][kpitch] (kpitch = n_out/64 rounded up to 4 for TMA): the same
// arithmetic as dq_decompress (doublequant.py:190-195), once per GEMM call.
__global__ void dq_constants_kernel(const uint8_t* __restrict__ dq_codes, const float* __restrict__ c1,
                                    const float* __restrict__ mu, int64_t rows, int64_t nbr, int64_t kpitch,
                                    int64_t ncols, int bs2, qlrt_fp8spec sp, float* __restrict__ out) {
  // columns [0, ncols) of each row (ncols = kpitch: the padding is zeroed;
  // ncols = nbr: one member's slice of a concatenated weight's cache)
  const float m = *mu;
  const int64_t total = rows * ncols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ncols, j = i - r * ncols;
    float c = 0.0f;
    if (j < nbr) {
      const int64_t blk = r * nbr + j;
      c = dq_constant(dq_codes[blk], c1[blk / bs2], m, sp);
    }
    out[r * kpitch + j] = c;
  }
}

// the block constants of up to 4 sibling weights (one row pitch, member g in
// columns [g nbr, (g + 1) nbr)) in one launch
struct GroupConsts {
  const uint8_t* dq_codes[4];
  const float* c1[4];
  const float* mu[4];
};
__global__ void dq_constants_group_kernel(GroupConsts gc, int groups, int64_t rows, int64_t nbr, int64_t kpitch,
                                          int bs2, qlrt_fp8spec sp, float* __restrict__ out) {
  const int64_t w = (int64_t)groups * nbr;
  const int64_t total = rows * w;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / w, jj = i - r * w;
    const int g = (int)(jj / nbr);
    const int64_t j = jj - (int64_t)g * nbr, blk = r * nbr + j;
    out[r * kpitch + jj] = dq_constant(gc.dq_codes[g][blk], gc.c1[g][blk / bs2], *gc.mu[g], sp);
  }
}

// many weights' block constants in one launch (blockIdx.y = job): the
// step-level prepass of a model's frozen linears
__global__ void dq_constants_batch_kernel(const qlrt_nf4_const_job* __restrict__ jobs) {
  const qlrt_nf4_const_job j = jobs[blockIdx.y];
  const float m = *j.mu;
  const int64_t total = j.rows * j.nbr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / j.nbr, c = i - r * j.nbr;
    j.out[r * j.pitch + c] = dq_constant(j.dq_codes[i], j.c1[i / j.blocksize2], m, j.spec);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// bf16 matrix stored row-major [outer][inner] with row pitch ld (elements);
// box = 64 inner x box_outer, 128B swizzle, out-of-bounds -> 0 (pads K, M, N).
static bool make_tmap(CUtensorMap* m, const void* base, int64_t inner, int64_t outer, int64_t ld, int box_outer) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || (((uintptr_t)base) & 15) || ((ld * 2) & 15)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// bf16 output written transposed by TMA stores: tensor [outer = N tokens][inner = M
// features] with row pitch ld, box 32 x 32, no swizzle (the epilogue's staging tile)
static bool make_tmap_store(CUtensorMap* m, const void* base, int64_t inner, int64_t outer, int64_t ld) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || (((uintptr_t)base) & 15) || ((ld * 2) & 15)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// packed NF4 codes viewed as a uint8 matrix [rows][bytes], no swizzle
static bool make_tmap_u8(CUtensorMap* m, const void* base, int64_t inner_bytes, int64_t rows, int box_inner,
                         int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || (((uintptr_t)base) & 15) || (inner_bytes & 15)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner_bytes, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)inner_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// One GEMM operand.  K-major: stored [rows][K] (pitch ld); MN-major: stored [K][rows].
struct Operand {
  const void* ptr = nullptr;
  int64_t ld = 0;
  int mn = 0;
};

// 2-CTA pairing policy: QLRT_PAIR=0 off, 1 on, unset -> the per-GEMM default
// Adapter product (Ts / dT) beside the fused GEMM that consumes it, chained by
// programmatic dependent launch (QLRT_OVERLAP=0 disables it): the skinny GEMM
// runs without split-K on `need` SMs while the fused grid starts its main K
// segment; only the fused grid's augmented loads wait for it.  Returns the
// pair cap for the fused grid (leaving >= need SMs), 0 when the cap would cost
// a round of 256 x 512 tiles -- then the old serial order is used.
static int overlap_cap(int64_t w_rows, int64_t m, int need_sms);
static int overlap_need_sms() { return policy(P_OVERLAP_SMS); }  // SMs left to the adapter product (8: +1-2% over 4)

static int pair_policy(int dflt) {
  const int v = policy(P_PAIR);
  return v < 0 ? dflt : v;
}

// A side stream (+ fork / join events) per (device, caller stream) for the
// independent skinny adapter GEMMs; QLRT_SIDE=0 keeps everything on the
// caller's stream.  Callers on different streams never share a side stream or
// its events; one caller's launches are ordered by its own stream.
struct SideCtx {
  int dev;
  cudaStream_t caller, side;
  cudaEvent_t ev[2];
};
static std::mutex g_side_mu;
static SideCtx g_side[256];
static int g_side_n = 0;
static SideCtx* side_ctx(cudaStream_t caller) {
  if (!policy(P_SIDE)) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_side_mu);
  for (int i = 0; i < g_side_n; ++i)
    if (g_side[i].dev == dev && g_side[i].caller == caller) return &g_side[i];
  if (g_side_n == 256) return nullptr;  // table full: the caller's stream only
  SideCtx c{dev, caller, nullptr, {nullptr, nullptr}};
  if (cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  if (cudaEventCreateWithFlags(&c.ev[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c.ev[1], cudaEventDisableTiming) != cudaSuccess)
    return nullptr;
  g_side[g_side_n] = c;
  return &g_side[g_side_n++];
}
static bool is_side_stream(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_side_mu);
  for (int i = 0; i < g_side_n; ++i)
    if (g_side[i].side == s) return true;
  return false;
}
// critical-path launches (the caller's stream) ahead of the side stream's
static void add_priority(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* attrs, cudaStream_t s) {
  const int pr = policy(P_PRIO);  // 1: the caller's stream first, 2: the side stream first
  if (!pr || is_side_stream(s) != (pr == 2)) return;
  cudaLaunchAttribute& at = attrs[cfg.numAttrs];
  at.id = cudaLaunchAttributePriority;
  at.val.priority = high_priority();
  cfg.attrs = attrs;
  cfg.numAttrs += 1;
}
// fork: the side stream waits for everything issued on `st` so far
static cudaStream_t fork_side(SideCtx* c, cudaStream_t st) {
  if (!c || cudaEventRecord(c->ev[0], st) != cudaSuccess || cudaStreamWaitEvent(c->side, c->ev[0], 0) != cudaSuccess)
    return nullptr;
  return c->side;
}
// join: `st` waits for everything issued on the side stream so far
static bool join_side(SideCtx* c, cudaStream_t st) {
  return cudaEventRecord(c->ev[1], c->side) == cudaSuccess && cudaStreamWaitEvent(st, c->ev[1], 0) == cudaSuccess;
}

// kernel attributes (dynamic shared memory) are per device: set once per device
static bool attr_once(std::atomic<unsigned long long>& mask, const void* kern, int bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  const unsigned long long bit = 1ull << dev;
  if (mask.load(std::memory_order_acquire) & bit) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  mask.fetch_or(bit, std::memory_order_acq_rel);
  return true;
}

// 256 x 512 pair tiles for the fused NF4 GEMMs (QLRT_TILE512=0 falls back to
// 128 x 256 single-CTA tiles): the 2-CTA pair halves the B traffic per SM and
// the two N = 256 UMMAs per k-step halve the dequant work per MMA -- measured
// +16..41% on the C2 / C4 shapes (tools/ab.py QLRT_TILE512=0/1)
static int tile512_policy() { return policy(P_TILE512); }

// per-half accumulator release for 512-wide tiles (QLRT_STAGGER=1).  Off by
// default: correct, but measured neutral-to-slower (tools/ab.py QLRT_STAGGER)
static int stagger_policy() { return policy(P_STAGGER); }

// epilogue output via TMA stores (QLRT_TMAOUT=0: ld.shared + 16 B st.global)
static int tma_out_policy() { return policy(P_TMAOUT); }

// half tiles for the last partial wave of 512-wide pair tiles (QLRT_HALFTAIL=0 disables)
static int halftail_policy() { return policy(P_HALFTAIL); }

// programmatic dependent launch of the engine kernels (QLRT_PDL=0 disables it)
static int pdl_policy() { return policy(P_PDL); }

// shared-decode CTA pairs for the fused NF4 GEMMs (QLRT_SHARE=1).  Off by
// default: correct, but the cross-SM coupling (both MMAs release a stage,
// both producer halves fill it, DSMEM stores + remote arrives) costs more
// than the halved decode saves -- measured 0.66x (tools/ab.py QLRT_SHARE=0/1)
static int share_policy() { return policy(P_SHARE); }

// stream-K policy: QLRT_STREAMK=0 disables it (whole-tile waves only)
static int streamk_policy() { return policy(P_STREAMK); }

static int num_sms();
static int overlap_cap(int64_t w_rows, int64_t m, int need_sms) {
  if (!policy(P_OVERLAP)) return 0;
  const int64_t tiles = ((w_rows + 255) / 256) * ((m + 511) / 512);
  auto rounds = [&](int64_t units) {
    const int64_t full = tiles / units, rem = tiles - full * units;
    return (double)full + (rem == 0 ? 0.0 : (2 * rem <= units && full > 0 ? 0.85 : 1.0));
  };
  const int64_t all = num_sms() / 2;
  int64_t cap = all - (need_sms + 1) / 2;
  if (tiles <= cap) return (int)tiles;  // the grid leaves enough SMs free already
  if (cap < 8 || rounds(cap) > rounds(all) + 1e-9) return 0;
  return (int)cap;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = kNumSMs;
  }
  return n;
}


template <int BN, bool NF4, bool PAIR = false>
static qlrt_status launch_t(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& a2, const CUtensorMap& b2,
                            const CUtensorMap& c, const CUtensorMap& k, const CUtensorMap& o, const Args& args,
                            cudaStream_t s) {
  using L = Smem<BN, NF4, PAIR>;
  auto kern = gemm_kernel<BN, NF4, PAIR>;
  static std::atomic<unsigned long long> attr_mask{0};
  if (!attr_once(attr_mask, (const void*)kern, L::BYTES)) return QLRT_ERR_CUDA;
  const int bmp = PAIR ? 2 * BM : BM;
  const int m_tiles = (args.M + bmp - 1) / bmp, n_tiles = (args.N + BN - 1) / BN;
  const int tiles = m_tiles * n_tiles * args.splits;
  int units_max = PAIR ? num_sms() / 2 : num_sms();
  if (args.units_cap > 0 && args.units_cap < units_max) units_max = args.units_cap;
  // stream-K: at most kSkMaxSplit units share a tile (the owner reads the
  // others' partials from L2; more contributors cost more round trips)
  int units = (tiles < units_max && !args.streamk) ? tiles : units_max;
  if (args.streamk && (int64_t)tiles * kSkMaxSplit < units) units = tiles * kSkMaxSplit;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(units * (PAIR ? 2 : 1));
  cfg.blockDim = dim3(NF4 ? kNF4Threads : kPlainThreads);
  cfg.dynamicSmemBytes = L::BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attrs[3];
  if (!PAIR && !NF4 && args.csplit > 1) {  // one CTA per (tile, split), clusters of csplit
    cfg.gridDim = dim3(m_tiles * n_tiles * args.csplit);
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = args.csplit;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
  }
  if (NF4 && !PAIR && args.share) {  // pairs of CTAs on the same W rows
    const int tiles_s = m_tiles * ((n_tiles + 1) / 2) * args.splits;
    const int pairs = tiles_s < num_sms() / 2 ? tiles_s : num_sms() / 2;
    cfg.gridDim = dim3(2 * pairs);
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = 2;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
  }
  if (!PAIR && !NF4 && args.cl2 && args.csplit <= 1) {
    cfg.gridDim = dim3((units + 1) / 2 * 2);
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = 2;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
  }
  if (PAIR) {
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = 2;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
  }
  if (pdl_policy()) {
    cudaLaunchAttribute& at = attrs[cfg.numAttrs];
    at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs += 1;
  }
  add_priority(cfg, attrs, s);
  if (cudaLaunchKernelEx(&cfg, kern, a, b, a2, b2, c, k, o, args) != cudaSuccess) return QLRT_ERR_CUDA;
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

static int effective_splits(int splits, int k_iters) {
  int sp = splits < 1 ? 1 : (splits > k_iters ? k_iters : splits);
  while (sp > 1 && (int64_t)(sp - 1) * ((k_iters + sp - 1) / sp) >= k_iters) --sp;  // every split owns >= 1 iter
  return sp;
}

// D[M,N] = A B (+ A2 B2).  K / K2 are true extents (TMA zero-fills the pad to 64).
// args.nf4_mode != 0 makes A the quantized weight (A operand ignored).
static qlrt_status run(int bn, const Operand& A, const Operand& B, const Operand* A2, const Operand* B2, int64_t K,
                       int64_t K2, Args args, cudaStream_t s) {
  CUtensorMap ta{}, tb{}, ta2{}, tb2{}, tc{}, tk{}, to{};
  const bool nf4 = args.nf4_mode != 0;
  if (nf4) {
    // packed codes as a uint8 matrix [w_rows][w_cols/2]; constants fp32 [w_rows][kpitch]
    const bool ok = args.nf4_mode == 1 ? make_tmap_u8(&tc, args.codes, args.w_cols / 2, args.w_rows, 64, 64)
                                       : make_tmap_u8(&tc, args.codes, args.w_cols / 2, args.w_rows, 32, 128);
    // the fp32 constants are moved as raw bytes (16 B = 4 floats per row)
    if (!ok || !make_tmap_u8(&tk, args.consts, args.kpitch * 4, args.w_rows, 16, args.nf4_mode == 1 ? 64 : 128))
      return QLRT_ERR_UNSUPPORTED;
    args.bs2_shift = (args.bs2 > 0 && (args.bs2 & (args.bs2 - 1)) == 0) ? __builtin_ctz((unsigned)args.bs2) : -1;
  } else {
    tc = tb;
    tk = tb;
  }
  const int64_t M = args.M, N = args.N;
  if (bn < 64 && (B.mn || (B2 && B2->mn))) return QLRT_ERR_UNSUPPORTED;
  const int64_t KA = args.kg_n ? args.kg_kfull : K;  // grouped-K: the operands' whole K extent
  if (args.kg_n && (nf4 || A.mn || B.mn || args.pair || bn % 64 || args.kg_n % bn || args.kg_k % BK))
    return QLRT_ERR_UNSUPPORTED;
  if (!nf4 && !(A.mn ? make_tmap(&ta, A.ptr, M, KA, A.ld, 64) : make_tmap(&ta, A.ptr, KA, M, A.ld, BM)))
    return QLRT_ERR_UNSUPPORTED;
  if (args.pair && ((bn != 256 && bn != 512) || (B2 && B2->mn && bn / 2 < 64))) return QLRT_ERR_UNSUPPORTED;
  if (bn == 512 && (!args.pair || B.mn || (B2 && B2->mn))) return QLRT_ERR_UNSUPPORTED;
  const int bbox = args.pair ? (bn > 256 ? 128 : bn / 2) : bn;  // B rows per TMA box
  if (!(B.mn ? make_tmap(&tb, B.ptr, N, KA, B.ld, 64)
             : make_tmap(&tb, B.ptr, KA, args.kg_n ? args.kg_n : N, B.ld, bbox)))
    return QLRT_ERR_UNSUPPORTED;
  if (K2) {
    const int64_t K2a = args.aug_wrap ? K2 / 2 : K2;  // A2's own K extent
    if (args.aug_wrap && (args.aug_wrap % BK || K2 % (2 * args.aug_wrap))) return QLRT_ERR_UNSUPPORTED;
    const int64_t K2b = args.aug_b2k > 0 ? args.aug_b2k : K2;
    if (!(A2->mn ? make_tmap(&ta2, A2->ptr, M, K2a, A2->ld, 64) : make_tmap(&ta2, A2->ptr, K2a, M, A2->ld, BM)))
      return QLRT_ERR_UNSUPPORTED;
    if (!(B2->mn ? make_tmap(&tb2, B2->ptr, N, K2b, B2->ld, 64) : make_tmap(&tb2, B2->ptr, K2b, N, B2->ld, bbox)))
      return QLRT_ERR_UNSUPPORTED;
  } else {
    ta2 = nf4 ? tb : ta;
    tb2 = tb;
  }
  args.k_iters = (int)((K + BK - 1) / BK);
  args.k_iters_aug = (int)((K2 + BK - 1) / BK);
  args.a_mn = A.mn;
  args.b_mn = B.mn;
  args.a2_mn = A2 ? A2->mn : 0;
  args.b2_mn = B2 ? B2->mn : 0;
  args.splits = effective_splits(args.splits, args.k_iters);
  if (args.csplit > 1) args.csplit = args.splits;  // every CTA of the cluster owns >= 1 k-iteration
  args.stagger = stagger_policy();
  args.tail_from = 0;
  if (bn == 512 && args.pair && !args.streamk && args.splits == 1 && halftail_policy()) {
    // whole 256 x 512 tiles for the full waves, half tiles for the last partial one
    const int64_t tiles = ((M + 255) / 256) * ((N + 511) / 512);
    const int64_t units = args.units_cap > 0 && args.units_cap < num_sms() / 2 ? args.units_cap : num_sms() / 2;
    const int64_t full = (tiles / units) * units;
    // a half tile costs ~0.85 of a whole one (same dequant): only worth it when
    // all the halves fit in one round
    if (full > 0 && full < tiles && 2 * (tiles - full) <= units) args.tail_from = (int)full;
  }
  if (args.splits > 1 && K2) return QLRT_ERR_UNSUPPORTED;
  // (not for the single-buffered 512-wide pair tiles: measured slower)
  if (args.sk_ws && args.splits == 1 && bn >= 64 && bn <= 256 && num_sms() <= kNumSMs && !args.share) {
    // stream-K only for short grids (< 2 waves) that whole-tile waves would
    // leave > 10% idle: measured, its partial-tile traffic and spread-out
    // L2 footprint cost ~5% on long grids (tools/ab.py QLRT_STREAMK=0/1)
    const int bmp = args.pair ? 2 * BM : BM;
    const int64_t tiles = ((M + bmp - 1) / bmp) * ((N + bn - 1) / bn);
    const int64_t units = args.pair ? num_sms() / 2 : num_sms();
    const int64_t waves = (tiles + units - 1) / units;
    const int64_t T = args.k_iters + args.k_iters_aug;
    args.streamk = waves <= 2 && (double)tiles / (double)(waves * units) < 0.9 && T * tiles >= 2 * units;
    if (args.aug_pdl || args.kg_n) args.streamk = 0;
    // the flags are zero between launches: every owner re-arms the flags it
    // consumed; the caller zero-fills the region once (qlrt_streamk_init)
  } else if (policy(P_SK512) > 0 && args.sk_ws && bn == 512 && args.pair && args.splits == 1 && !args.aug_pdl &&
             !args.kg_n && !args.share) {
    // QLRT_SK512 = min k-iterations: stream-K over 256 x 512 pair tiles for a
    // grid of fewer tiles than SM pairs (one partial round) with a long K
    // loop -- every pair gets ~tiles / pairs of the K work, partial tiles
    // fixed up through the stream-K region
    const int64_t tiles = ((M + 255) / 256) * ((N + 511) / 512);
    const int64_t units = args.units_cap > 0 && args.units_cap < num_sms() / 2 ? args.units_cap : num_sms() / 2;
    const int64_t T = args.k_iters + args.k_iters_aug;
    args.streamk = tiles < units && T >= policy(P_SK512) && num_sms() <= kNumSMs;
    if (args.streamk) args.tail_from = 0;
  } else {
    args.streamk = 0;
  }
  // bf16 D^T output through TMA stores (32 features x 32 tokens per box)
  args.tma_out = 0;
  if (args.out_t && !args.out_f32 && args.splits == 1 && !args.to_ws && !args.out_split && tma_out_policy() &&
      make_tmap_store(&to, args.out, args.M, args.N, args.ldo))
    args.tma_out = 1;
  if (!args.tma_out) to = tb;
  args.pdl_trigger = policy(P_PDL_TRIGGER) && pdl_policy() && (!args.aug_pdl || args.trigger_dep);
  switch (bn) {
    case 512:
      return nf4 ? launch_t<512, true, true>(ta, tb, ta2, tb2, tc, tk, to, args, s)
                 : launch_t<512, false, true>(ta, tb, ta2, tb2, tc, tk, to, args, s);
    case 256:
      if (args.pair) return nf4 ? launch_t<256, true, true>(ta, tb, ta2, tb2, tc, tk, to, args, s)
                                : launch_t<256, false, true>(ta, tb, ta2, tb2, tc, tk, to, args, s);
      return nf4 ? launch_t<256, true>(ta, tb, ta2, tb2, tc, tk, to, args, s) : launch_t<256, false>(ta, tb, ta2, tb2, tc, tk, to, args, s);
    case 128: return nf4 ? launch_t<128, true>(ta, tb, ta2, tb2, tc, tk, to, args, s) : launch_t<128, false>(ta, tb, ta2, tb2, tc, tk, to, args, s);
    case 64: return nf4 ? launch_t<64, true>(ta, tb, ta2, tb2, tc, tk, to, args, s) : launch_t<64, false>(ta, tb, ta2, tb2, tc, tk, to, args, s);
    case 16: return nf4 ? launch_t<16, true>(ta, tb, ta2, tb2, tc, tk, to, args, s) : launch_t<16, false>(ta, tb, ta2, tb2, tc, tk, to, args, s);
  }
  return QLRT_ERR_UNSUPPORTED;
}

static qlrt_status reduce(const Args& args, cudaStream_t s) {
  const int64_t total = (int64_t)args.M * (args.fold ? args.N / 2 : args.N);
  int64_t g = (total + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)g);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  if (pdl_policy()) {  // launched early behind the split-K GEMM (see Args::pdl_trigger)
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  add_priority(cfg, at, s);
  if (cudaLaunchKernelEx(&cfg, splitk_reduce_kernel, (const float*)args.ws, args.splits, args.M, args.N, args.fold,
                         args.alpha, args.out, args.ldo, args.out_f32, args.out_t, args.out_split) != cudaSuccess)
    return QLRT_ERR_CUDA;
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

// split count that fills the machine for a tile grid, bounded by workspace
static int pick_splits(int64_t tiles, int64_t k_iters, int64_t per_split_bytes, size_t ws_bytes) {
  if (tiles >= 74 || k_iters < 8) return 1;
  // CTA budget (QLRT_SKINNY_CTAS): 148 = one per SM; the 64-wide skinny
  // GEMMs fit two per SM (4 stages of 24 KB each)
  int64_t sp = policy(P_SKINNY_CTAS) / tiles;
  if (sp > k_iters / 4) sp = k_iters / 4;
  if (sp > 16) sp = 16;
  if (per_split_bytes > 0 && (int64_t)ws_bytes / per_split_bytes < sp) sp = (int64_t)ws_bytes / per_split_bytes;
  return sp < 1 ? 1 : (int)sp;
}

// D = alpha A B with automatic split-K (skinny LoRA GEMMs).  fold: see the
// reduce kernel (forces the fp32 workspace route); out_split: bf16 hi/lo.
static qlrt_status plain(int bn, const Operand& A, const Operand& B, int64_t M, int64_t N, int64_t K, float alpha,
                         void* out, int64_t ldo, int out_f32, int out_t, float* ws, size_t ws_bytes, cudaStream_t s,
                         int fold = 0, int out_split = 0, const Args* sk = nullptr, int pdl_independent = 0,
                         int cl2 = 0, int units_cap = 0, int kg_n = 0, int64_t kg_kfull = 0) {
  Args a{};
  a.cl2 = cl2;
  a.units_cap = units_cap;
  a.kg_n = kg_n;  // grouped-K (see Args): member width along N, K = one member's K extent
  a.kg_k = kg_n ? K : 0;
  a.kg_kfull = kg_kfull;
  // pdl_independent: inputs only (nothing from the PDL predecessor) -- start
  // at once beside it, complete only after it (see Args::wait_at_end)
  a.aug_pdl = pdl_independent;
  a.wait_at_end = pdl_independent;
  a.M = (int)M;
  a.N = (int)N;
  a.out = out;
  a.ldo = ldo;
  a.out_f32 = out_f32;
  a.out_t = out_t;
  a.alpha = alpha;
  a.ws = ws;
  a.bs2 = 1;
  a.fold = fold;
  a.out_split = out_split;
  a.pair = (bn == 256 && !B.mn) ? pair_policy(1) : 0;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
  const int64_t kit = (K + BK - 1) / BK;
  // (off by default: measured slower than split-K + reduce on the C2 LoRA shapes,
  //  tools/ab_skinny.py; QLRT_STREAMK_SKINNY=1 enables it)
  if (policy(P_STREAMK_SKINNY) && !kg_n && sk && sk->sk_ws && streamk_policy() && !(out_split && out_t) &&
      (!fold || (2 * fold <= bn && N <= bn))) {
    // skinny GEMM: stream-K over all SMs, partials reduced in-kernel, fold /
    // hi-lo split applied in the epilogue -- no split-K workspace, no reduce launch
    a.sk_ws = sk->sk_ws;
    a.sk_flags = sk->sk_flags;
    a.splits = 1;
    a.to_ws = 0;
    return run(bn, A, B, nullptr, nullptr, K, 0, a, s);
  }
  // cluster split-K for short grids: partials reduced over DSMEM inside the
  // kernel.  Off by default (QLRT_CSPLIT=1 enables it): measured 1.7-2.9x
  // slower than split-K + the reduce kernel on the C2 LoRA shapes
  // (tools/ab_skinny.py) -- clusters of 1-CTA-per-SM kernels co-schedule poorly
  if (policy(P_CSPLIT) && !kg_n && tiles < 74 && !(out_split && out_t) && bn <= 256 && a.pair == 0 &&
      (!fold || (2 * fold <= bn && N <= bn))) {
    int S = 1;
    while (S < 8 && tiles * (S + 1) <= num_sms() && (S + 1) * 4 <= kit) ++S;
    if (S >= 2) {
      a.splits = S;
      a.csplit = S;
      a.to_ws = 0;
      return run(bn, A, B, nullptr, nullptr, K, 0, a, s);
    }
  }
  a.splits = effective_splits(ws ? pick_splits(tiles, kit, M * N * 4, ws_bytes) : 1, (int)kit);
  // fold is applied in the epilogue when one column tile holds both halves
  // and there is no split-K (no reduce launch); otherwise the reduce kernel folds
  const bool direct_fold = fold != 0 && a.splits == 1 && 2 * fold <= bn && N == 2 * fold;
  a.to_ws = (fold != 0 && !direct_fold) || (out_split && out_t);
  if ((a.to_ws || a.splits > 1) && (!ws || (size_t)(M * N * 4) * a.splits > ws_bytes)) return QLRT_ERR_ARG;
  qlrt_status st = run(bn, A, B, nullptr, nullptr, K, 0, a, s);
  if (st != QLRT_OK || (a.splits == 1 && !a.to_ws)) return st;
  return reduce(a, s);
}

static int64_t kpitch_of(const qlrt_nf4_weight* w) { return ((w->n_out / 64) + 3) / 4 * 4; }
static size_t consts_bytes(int64_t k_in, int64_t n_out) {
  return (size_t)k_in * (size_t)(((n_out / 64) + 3) / 4 * 4) * 4;
}

// NF4 operand description + the per-call constants prepass into `consts`
static qlrt_status fill_nf4(Args& a, const qlrt_nf4_weight* w, int mode, float* consts, cudaStream_t st) {
  a.nf4_mode = mode;
  a.codes = w->codes;
  a.dq_codes = w->dq_codes;
  a.c1 = w->c1;
  a.mu = w->mu;
  a.absmax = nullptr;
  a.w_rows = w->k_in;
  a.w_cols = w->n_out;
  a.bs2 = w->blocksize2;
  a.spec = w->spec;
  for (int i = 0; i < 16; ++i) a.values[i] = w->values[i];
  a.kpitch = kpitch_of(w);
  if (w->consts) {  // caller-provided cache, already filled by qlrt_nf4_constants
    a.consts = w->consts;
    return QLRT_OK;
  }
  a.consts = consts;
  const int64_t total = w->k_in * a.kpitch;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  dq_constants_kernel<<<(int)g, 256, 0, st>>>(w->dq_codes, w->c1, w->mu, w->k_in, w->n_out / 64, a.kpitch, a.kpitch,
                                             w->blocksize2, w->spec, consts);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

static bool weight_ok(const qlrt_nf4_weight* w) {
  return w && w->codes && w->dq_codes && w->c1 && w->mu && w->k_in > 0 && w->n_out > 0 && (w->n_out % 64) == 0 &&
         (((uintptr_t)w->codes) & 15) == 0 && w->blocksize2 > 0;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// bytes of the doubled adapter operand ([l1|l1] or [l2;l2], bf16)
static size_t dbl_bytes(int64_t k_in, int64_t n_out, int rank) {
  const int64_t mx = k_in > n_out ? k_in : n_out;
  return align256((size_t)mx * 2 * rank * 2);
}
// split-K partial bytes of one skinny adapter GEMM (<= 16 splits)
static size_t side_part_bytes(int64_t m, int64_t k_in, int64_t n_out, int rank) {
  const int64_t r = rank > 0 ? rank : 1;
  int64_t a = 16 * m * 2 * r, b = 16 * k_in * 2 * r, c = 16 * 2 * r * n_out;
  int64_t mx = a > b ? a : b;
  mx = mx > c ? mx : c;
  return align256((size_t)mx * 4);
}
// stream-K partials (one BM x 256 fp32 tile per CTA) + flags
constexpr int kSkCols = 512;  // widest tile (pair 256 x 512)
static size_t sk_bytes() { return align256((size_t)kNumSMs * BM * kSkCols * 4) + align256((size_t)kNumSMs * 4); }
// layout of the linear workspace: [split-K partials][constants][stream-K][doubled adapter]
static void* dbl_region(void* ws, size_t ws_bytes, int64_t k_in, int64_t n_out, int rank) {
  return (uint8_t*)ws + (ws_bytes - dbl_bytes(k_in, n_out, rank));
}
static void sk_region(void* ws, size_t ws_bytes, int64_t k_in, int64_t n_out, int rank, Args& a) {
  uint8_t* b = (uint8_t*)ws + (ws_bytes - dbl_bytes(k_in, n_out, rank) - sk_bytes());
  a.sk_ws = (float*)b;
  a.sk_flags = (int*)(b + align256((size_t)kNumSMs * BM * kSkCols * 4));
}

}  // namespace gemm
}  // namespace qlrt

using namespace qlrt;
using gemm::Operand;

extern "C" {

#ifdef QLRT_TRACE
// copies and clears the per-CTA trace totals ([2 * 148][24] u64)
int qlrt_trace_fetch(unsigned long long* host) {
  static unsigned long long zero[2 * qlrt::kNumSMs][qlrt::gemm::kTrSlots];
  if (cudaMemcpyFromSymbol(host, qlrt::gemm::g_trace, sizeof(zero)) != cudaSuccess) return -1;
  return cudaMemcpyToSymbol(qlrt::gemm::g_trace, zero, sizeof(zero)) == cudaSuccess ? 0 : -1;
}
#endif

int qlrt_set_policy(const char* name, int value) {
  if (!name) return QLRT_ERR_ARG;
  if (!g_policy_init.load(std::memory_order_acquire)) policy_load_env();
  for (int i = 0; i < P_COUNT; ++i)
    if (!strcmp(name, kPolicies[i].env)) {
      g_policy[i].store(value == kPolicyUnset ? kPolicies[i].dflt : value, std::memory_order_relaxed);
      return QLRT_OK;
    }
  return QLRT_ERR_ARG;
}

int qlrt_get_policy(const char* name, int* value) {
  if (!name || !value) return QLRT_ERR_ARG;
  for (int i = 0; i < P_COUNT; ++i)
    if (!strcmp(name, kPolicies[i].env)) {
      *value = policy((Policy)i);
      return QLRT_OK;
    }
  return QLRT_ERR_ARG;
}

size_t qlrt_nf4_constants_bytes(int64_t k_in, int64_t n_out) { return gemm::consts_bytes(k_in, n_out); }

qlrt_status qlrt_nf4_constants(const qlrt_nf4_weight* w, float* out, void* stream) {
  if (!w || !w->dq_codes || !w->c1 || !w->mu || !out || w->n_out % 64) return QLRT_ERR_ARG;
  qlrt_nf4_weight tmp = *w;
  tmp.consts = nullptr;
  gemm::Args a{};
  return gemm::fill_nf4(a, &tmp, 1, out, (cudaStream_t)stream);
}

qlrt_status qlrt_nf4_constants_into(const qlrt_nf4_weight* w, float* out, int64_t pitch, void* stream) {
  // one member's block constants into columns [0, n_out / 64) of rows of
  // `pitch` floats (out = the member's first column of a concatenated cache)
  if (!w || !w->dq_codes || !w->c1 || !w->mu || !out || w->n_out % 64 || pitch < w->n_out / 64 ||
      w->blocksize2 <= 0)
    return QLRT_ERR_ARG;
  const int64_t nbr = w->n_out / 64;
  int64_t g = (w->k_in * nbr + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  gemm::dq_constants_kernel<<<(int)g, 256, 0, (cudaStream_t)stream>>>(w->dq_codes, w->c1, w->mu, w->k_in, nbr, pitch,
                                                                      nbr, w->blocksize2, w->spec, out);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_nf4_constants_group(const qlrt_nf4_weight* members, int groups, float* out, int64_t pitch,
                                     void* stream) {
  // every member's constants into one concatenated cache (one launch)
  if (!members || groups < 1 || groups > 4 || !out) return QLRT_ERR_ARG;
  gemm::GroupConsts gc{};
  for (int g = 0; g < groups; ++g) {
    const qlrt_nf4_weight& w = members[g];
    if (!w.dq_codes || !w.c1 || !w.mu || w.n_out % 64 || w.k_in != members[0].k_in || w.n_out != members[0].n_out ||
        w.blocksize2 != members[0].blocksize2 || w.blocksize2 <= 0)
      return QLRT_ERR_ARG;
    gc.dq_codes[g] = w.dq_codes;
    gc.c1[g] = w.c1;
    gc.mu[g] = w.mu;
  }
  const int64_t nbr = members[0].n_out / 64;
  if (pitch < groups * nbr) return QLRT_ERR_ARG;
  int64_t g = (members[0].k_in * groups * nbr + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  gemm::dq_constants_group_kernel<<<(int)g, 256, 0, (cudaStream_t)stream>>>(
      gc, groups, members[0].k_in, nbr, pitch, members[0].blocksize2, members[0].spec, out);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

qlrt_status qlrt_nf4_constants_batch(const qlrt_nf4_const_job* jobs_dev, int n_jobs, int64_t max_elems,
                                     void* stream) {
  if (!jobs_dev || n_jobs < 1 || n_jobs > 65535 || max_elems < 1) return QLRT_ERR_ARG;
  int64_t gx = (max_elems + 255) / 256;
  if (gx > 64) gx = 64;  // (grid-stride: n_jobs x 64 CTAs keep every SM busy)
  gemm::dq_constants_batch_kernel<<<dim3((unsigned)gx, (unsigned)n_jobs), 256, 0, (cudaStream_t)stream>>>(jobs_dev);
  QLRT_CHECK_LAUNCH();
  return QLRT_OK;
}

size_t qlrt_linear_workspace_bytes(int64_t m, int64_t k_in, int64_t n_out, int rank) {
  // split-K partials of the skinny adapter GEMMs (<= 16 splits each) + GEMV scratch
  size_t total = gemm::side_part_bytes(m, k_in, n_out, rank) + 4096 +
                 gemm::align256(gemm::consts_bytes(k_in, n_out)) + gemm::sk_bytes() +
                 gemm::dbl_bytes(k_in, n_out, rank > 0 ? rank : 0);
  const size_t gv = qlrt_gemv_workspace_bytes(k_in, n_out, rank > 0 ? rank : 0);  // M = 1 path
  return total > gv ? total : gv;
}

qlrt_status qlrt_gemm_bf16(const void* a, const void* b, void* d, int64_t m, int64_t n, int64_t k, int a_mn, int b_mn,
                           float alpha, int out_f32, int out_t, void* workspace, size_t workspace_bytes, void* stream) {
  if (!a || !b || !d || m <= 0 || n <= 0 || k <= 0) return QLRT_ERR_ARG;
  Operand A, B;
  A.ptr = a; A.mn = a_mn; A.ld = a_mn ? m : k;
  B.ptr = b; B.mn = b_mn; B.ld = b_mn ? n : k;
  const int bn = n <= 64 ? 64 : (n <= 128 ? 128 : 256);
  // a workspace with room for the stream-K region (its last sk_bytes) enables stream-K
  gemm::Args sk{};
  if (workspace && workspace_bytes >= gemm::sk_bytes() + 4096) {
    uint8_t* b = (uint8_t*)workspace + (workspace_bytes - gemm::sk_bytes());
    b = (uint8_t*)(((uintptr_t)b) & ~(uintptr_t)255);
    sk.sk_ws = (float*)b;
    sk.sk_flags = (int*)(b + gemm::align256((size_t)kNumSMs * gemm::BM * gemm::kSkCols * 4));
    workspace_bytes = (size_t)(b - (uint8_t*)workspace);
  }
  return gemm::plain(bn, A, B, m, n, k, alpha, d, out_t ? m : n, out_f32, out_t, (float*)workspace, workspace_bytes,
                     (cudaStream_t)stream, 0, 0, sk.sk_ws ? &sk : nullptr);
}

qlrt_status qlrt_nf4_linear_fwd(const qlrt_nf4_weight* w, const void* x, const void* xa, int64_t m, const void* l1,
                                const void* l2, int rank, float s, void* ts_out, void* y, void* workspace,
                                void* stream) {
  if (!gemm::weight_ok(w) || !x || !y || m <= 0 || rank < 0) return QLRT_ERR_ARG;
  if (rank > 0 && (!l2 || !ts_out || (rank % 8))) return QLRT_ERR_ARG;
  // l1 == NULL: ts_out already holds Ts (several adapters concatenated by the host)
  const bool ts_given = rank > 0 && !l1;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t K = w->k_in, N = w->n_out;
  const size_t ws_bytes = qlrt_linear_workspace_bytes(m, K, N, rank);
  const size_t part_bytes =
      ws_bytes - gemm::dbl_bytes(K, N, rank) - gemm::sk_bytes() - gemm::align256(gemm::consts_bytes(K, N));
  float* consts = (float*)((uint8_t*)workspace + part_bytes);
  qlrt_status rc;
  gemm::Args sk{};
  gemm::sk_region(workspace, ws_bytes, K, N, rank, sk);
  const bool big = gemm::tile512_policy();
  const int cap = (rank > 0 && !ts_given && rank % 64 == 0 && big && gemm::pdl_policy())
                      ? gemm::overlap_cap(N, m, (policy(P_CL2) & 1) ? (int)((cdiv(m, 128) + 1) / 2 * 2) : gemm::overlap_need_sms())
                      : 0;
  if (cap) {
    // Ts beside the fused grid: constants first (the fused grid reads them from
    // its start), then Ts without split-K (bf16 hi/lo pair, one CTA per 128
    // tokens) as the PDL predecessor of the fused GEMM, whose TMA producer
    // waits for it only before the augmented segment [l2 ; l2]^T [Ts_hi | Ts_lo]^T
    gemm::Args a{};
    if ((rc = gemm::fill_nf4(a, w, 1, consts, st)) != QLRT_OK) return rc;
    Operand TA{xa ? xa : x, K, 0}, TB{l1, rank, 1};
    // (one CTA per 128-token tile; capping it to the SMs left, each CTA
    // looping over tiles, was measured slower: Ts then outlasts the grid's
    // first tiles)
    rc = gemm::plain(64, TA, TB, m, rank, K, s, ts_out, 2 * rank, 0, 0, nullptr, 0, st, 0, rank, nullptr, 0,
                     policy(P_CL2) & 1);
    if (rc != QLRT_OK) return rc;
    a.M = (int)N;
    a.N = (int)m;
    a.splits = 1;
    a.out = y;
    a.ldo = N;
    a.out_t = 1;
    a.alpha = 1.0f;
    a.pair = 1;
    a.aug_wrap = rank;
    a.aug_pdl = 1;
    a.units_cap = cap;
    Operand none{}, B{x, K, 0}, A2{l2, N, 1}, B2{ts_out, 2 * rank, 0};
    return gemm::run(512, none, B, &A2, &B2, K, 2 * rank, a, st);
  }
  // the block-constant prepass (when no cache is given) and the doubled l2
  // copies run on the side stream while Ts is computed here
  gemm::Args a{};
  gemm::SideCtx* sctx = rank > 0 ? gemm::side_ctx(st) : nullptr;
  cudaStream_t side = gemm::fork_side(sctx, st);
  cudaStream_t aux = side ? side : st;
  if ((rc = gemm::fill_nf4(a, w, 1, consts, aux)) != QLRT_OK) return rc;
  __nv_bfloat16* l2d = (__nv_bfloat16*)gemm::dbl_region(workspace, ws_bytes, K, N, rank);
  // rank % 64 == 0: the augmented operand re-reads l2 itself (no doubled copy)
  const bool wrap = rank > 0 && rank % 64 == 0;
  if (rank && !wrap) {
    if (cudaMemcpyAsync(l2d, l2, (size_t)rank * N * 2, cudaMemcpyDeviceToDevice, aux) != cudaSuccess ||
        cudaMemcpyAsync(l2d + (size_t)rank * N, l2, (size_t)rank * N * 2, cudaMemcpyDeviceToDevice, aux) != cudaSuccess)
      return QLRT_ERR_CUDA;
  }
  if (rank > 0 && !ts_given) {
    // Ts[m, 0:r] + Ts[m, r:2r] = s * Xa l1 as a bf16 hi/lo pair:
    //   A = Xa (K-major, [m][K]), B = l1 (MN-major, [K][r])
    Operand A{xa ? xa : x, K, 0}, B{l1, rank, 1};
    rc = gemm::plain(64, A, B, m, rank, K, s, ts_out, 2 * rank, 0, 0, (float*)workspace, part_bytes, st, 0, rank,
                     &sk);
    if (rc != QLRT_OK) return rc;
  }
  if (side && !gemm::join_side(sctx, st)) return QLRT_ERR_CUDA;
  // Y^T[N, m] = W^T X^T (+ l2^T Ts^T): A = NF4 (MN-major image), B = X (K-major)
  a.M = (int)N;
  a.N = (int)m;
  a.splits = 1;
  a.out = y;
  a.ldo = N;
  a.out_f32 = 0;
  a.out_t = 1;
  a.alpha = 1.0f;
  const int bn_main = gemm::tile512_policy() ? 512 : 256;
  a.pair = bn_main == 512 ? 1 : gemm::pair_policy(0);
  a.share = a.pair ? 0 : gemm::share_policy();
  if (gemm::streamk_policy()) { a.sk_ws = sk.sk_ws; a.sk_flags = sk.sk_flags; }
  Operand none{}, B{x, K, 0};
  // augmented segment K2 = 2r: [l2 ; l2]^T [Ts_hi | Ts_lo]^T, i.e. the pair at ~16-bit precision
  Operand A2{wrap ? l2 : l2d, N, 1}, B2{ts_out, 2 * rank, 0};
  a.aug_wrap = wrap ? rank : 0;
  return gemm::run(bn_main, none, B, rank ? &A2 : nullptr, rank ? &B2 : nullptr, K, 2 * rank, a, st);
}

qlrt_status qlrt_nf4_linear_bwd_ex(const qlrt_nf4_weight* w, const void* dy, int64_t m, const void* x,
                                   const void* ts, const void* l1, const void* l2, int rank, float s, void* dt_out,
                                   void* dx, float* dl1, float* dl2, void* workspace, void* side_workspace,
                                   int flags, void* stream) {
  if (!gemm::weight_ok(w) || !dy || !dx || m <= 0 || rank < 0 || (flags & ~QLRT_BWD_DEFER)) return QLRT_ERR_ARG;
  if (rank > 0 && (!x || !ts || !l1 || !dt_out || !dl1 || !dl2 || (rank % 8))) return QLRT_ERR_ARG;
  // l2 == NULL: dt_out already holds dT (several adapters concatenated by the host)
  const bool dt_given = rank > 0 && !l2;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t K = w->k_in, N = w->n_out;
  const size_t ws_bytes = qlrt_linear_workspace_bytes(m, K, N, rank);
  const size_t part_bytes =
      ws_bytes - gemm::dbl_bytes(K, N, rank) - gemm::sk_bytes() - gemm::align256(gemm::consts_bytes(K, N));
  float* consts = (float*)((uint8_t*)workspace + part_bytes);
  qlrt_status rc;
  gemm::Args sk{};
  gemm::sk_region(workspace, ws_bytes, K, N, rank, sk);
  // QLRT_BWD_DEFER: the adapter-gradient GEMMs (dl2, dl1) stay on the side
  // stream, not joined -- they run beside whatever the caller issues next
  // (the next layers' fused grids leave SMs idle) until qlrt_side_join.  Their
  // split-K partials then live in side_workspace (the caller's next calls reuse
  // `workspace` on its own stream meanwhile).
  gemm::SideCtx* sctx = rank > 0 ? gemm::side_ctx(st) : nullptr;
  const bool defer = (flags & QLRT_BWD_DEFER) && rank > 0 && sctx && side_workspace;
  const int side_cap = defer ? (policy(P_SIDE_SMS) + 0) : 0;  // units cap of the deferred GEMMs (0: none)
  const int bn_g = 2 * rank <= 64 ? 64 : (2 * rank <= 128 ? 128 : 256);
  // QLRT_OVERLAP_BWD=1: dT beside the fused dX grid as its PDL predecessor
  // (no split-K; the grid waits for it only before the augmented segment).
  // Without deferral it measured -6% to +2% (dl2 / dl1 then trail the grid at
  // full width); the 16 dT CTAs land one per SM and hold back fused pairs
  // that need whole SMs unless they run as 2-CTA clusters (QLRT_CL2 & 2).
  const int cap = (policy(P_OVERLAP_BWD) && rank > 0 && !dt_given && rank % 64 == 0 && gemm::tile512_policy() &&
                   gemm::pdl_policy())
                      ? gemm::overlap_cap(K, m, (policy(P_CL2) & 2) ? (int)((cdiv(m, 128) + 1) / 2 * 2) : gemm::overlap_need_sms())
                      : 0;
  const int diag = policy(P_DIAG_SKIP);
  gemm::Args a{};
  a.M = (int)K;
  a.N = (int)m;
  a.splits = 1;
  a.out = dx;
  a.ldo = K;
  a.out_f32 = 0;
  a.out_t = 1;
  a.alpha = 1.0f;
  Operand none{}, B{dy, N, 0};
  cudaStream_t side = nullptr;
  if (cap) {
    if ((rc = gemm::fill_nf4(a, w, 2, consts, st)) != QLRT_OK) return rc;
    Operand DA{dy, N, 0}, DB{l2, N, 0};
    rc = gemm::plain(64, DA, DB, m, rank, N, s, dt_out, 2 * rank, 0, 0, nullptr, 0, st, 0, rank, nullptr, 0,
                     (policy(P_CL2) >> 1) & 1);
    if (rc != QLRT_OK) return rc;
    a.pair = 1;
    a.aug_wrap = rank;
    a.aug_pdl = 1;
    a.units_cap = cap;
    Operand A2{l1, rank, 0}, B2{dt_out, 2 * rank, 0};
    // (dl2 / dl1 wait for dT: fork before the fused grid is issued, after dT)
    side = gemm::fork_side(sctx, st);
    if ((rc = gemm::run(512, none, B, &A2, &B2, N, 2 * rank, a, st)) != QLRT_OK) return rc;
  } else {
    if (rank > 0 && !dt_given && !(diag & 2)) {
      // dT[m, 0:r] + dT[m, r:2r] = s * dY l2^T (bf16 hi/lo pair):
      //   A = dY (K-major [m][N]), B = l2 (K-major [r][N])
      Operand DA{dy, N, 0}, DB{l2, N, 0};
      rc = gemm::plain(64, DA, DB, m, rank, N, s, dt_out, 2 * rank, 0, 0, (float*)workspace, part_bytes, st, 0, rank,
                       &sk);
      if (rc != QLRT_OK) return rc;
    }
    // the adapter gradients dl2 and dl1 need only the inputs and dT: they run on
    // a side stream forked here and are launched after the fused dX GEMM, so
    // they fill the SMs its grid leaves idle (or follow it as its CTAs retire)
    side = gemm::fork_side(sctx, st);
    // dX^T[K, m] = W dY^T (+ l1 dT^T): A = NF4 (K-major image), B = dY (K-major)
    const int bn_main = gemm::tile512_policy() ? 512 : 256;
    a.pair = bn_main == 512 ? 1 : gemm::pair_policy(0);
    a.share = a.pair ? 0 : gemm::share_policy();
    if (gemm::streamk_policy()) { a.sk_ws = sk.sk_ws; a.sk_flags = sk.sk_flags; }
    if ((rc = gemm::fill_nf4(a, w, 2, consts, st)) != QLRT_OK) return rc;
    // augmented segment K2 = 2r: [l1 | l1] [dT_hi | dT_lo]^T
    __nv_bfloat16* l1d = (__nv_bfloat16*)gemm::dbl_region(workspace, ws_bytes, K, N, rank);
    const bool wrap = rank > 0 && rank % 64 == 0;  // re-read l1 itself (no doubled copy)
    if (rank && !wrap) {
      for (int h = 0; h < 2; ++h)
        if (cudaMemcpy2DAsync(l1d + h * rank, (size_t)4 * rank, l1, (size_t)2 * rank, (size_t)2 * rank, (size_t)K,
                              cudaMemcpyDeviceToDevice, st) != cudaSuccess)
          return QLRT_ERR_CUDA;
    }
    Operand A2{wrap ? l1 : l1d, wrap ? rank : 2 * rank, 0}, B2{dt_out, 2 * rank, 0};
    a.aug_wrap = wrap ? rank : 0;
    rc = gemm::run(bn_main, none, B, rank ? &A2 : nullptr, rank ? &B2 : nullptr, N, 2 * rank, a, st);
    if (rc != QLRT_OK || rank == 0) return rc;
  }
  if (diag & 1) return side && !defer && !gemm::join_side(sctx, st) ? QLRT_ERR_CUDA : QLRT_OK;
  cudaStream_t aux = side ? side : st;
  {
    // dl2^T[N, r] = dY^T (Ts_hi + Ts_lo): A = dY (MN-major [m][N]), B = [Ts_hi | Ts_lo]
    // (MN-major [m][2r]); the pair is folded in the epilogue, stored transposed
    // into dl2[r][N] (no split-K: the workspace belongs to dl1)
    Operand A{dy, N, 1}, B2t{ts, 2 * rank, 1};
    rc = gemm::plain(bn_g, A, B2t, N, 2 * rank, m, 1.0f, dl2, N, 1, 1, nullptr, 0, aux, rank, 0, nullptr, 0, 0,
                     side_cap);
    if (rc != QLRT_OK) return rc;
  }
  {
    // dl1[K, r] = Xa^T (dT_hi + dT_lo): A = Xa (MN-major [m][K]), B = [dT_hi | dT_lo] (MN-major [m][2r])
    // (on the side stream it runs beside the fused dX grid, which owns the
    // stream-K region: no stream-K for it there; deferred, its split-K
    // partials go to the side workspace)
    Operand A{x, K, 1}, B1{dt_out, 2 * rank, 1};
    float* pw = defer ? (float*)side_workspace : (float*)workspace;
    rc = gemm::plain(bn_g, A, B1, K, 2 * rank, m, 1.0f, dl1, rank, 1, 0, pw, part_bytes, aux, rank, 0,
                     side ? nullptr : &sk, 0, 0, side_cap);
    if (rc != QLRT_OK) return rc;
  }
  if (side && !defer && !gemm::join_side(sctx, st)) return QLRT_ERR_CUDA;
  return rc;
}

// ---- sibling projections concatenated along N (q | k | v, gate | up) --------
// W_cat = [W_0 | ... | W_{G-1}] with N_g = n_out / G columns each (N_g % 256
// == 0: a 256-row tile of the fused GEMM never straddles two members), the
// block-constant cache w->consts filled per member (column slices), one
// adapter of rank r (r % 64 == 0) per member: l1_cat [K][G r], l2_cat [r][N].
// Ts_cat / dT_cat hold each member's bf16 [hi | lo] pair: [m][G 2r].
static bool group_ok(const qlrt_nf4_weight* w, int groups, int rank) {
  return gemm::weight_ok(w) && w->consts && groups >= 1 && w->n_out % groups == 0 &&
         (w->n_out / groups) % 256 == 0 && rank > 0 && rank % 64 == 0;
}

qlrt_status qlrt_nf4_linear_group_fwd(const qlrt_nf4_weight* w, int groups, const void* x, int64_t m,
                                      const void* l1, const void* l2, int rank, float s, void* ts_out, void* y,
                                      void* workspace, void* stream) {
  if (!group_ok(w, groups, rank) || !x || !y || !l1 || !l2 || !ts_out || !workspace || m <= 0) return QLRT_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t K = w->k_in, N = w->n_out, Ng = N / groups;
  const int R = groups * rank;
  const size_t ws_bytes = qlrt_linear_workspace_bytes(m, K, N, R);
  const size_t part_bytes =
      ws_bytes - gemm::dbl_bytes(K, N, R) - gemm::sk_bytes() - gemm::align256(gemm::consts_bytes(K, N));
  gemm::Args sk{};
  gemm::sk_region(workspace, ws_bytes, K, N, R, sk);
  qlrt_status rc;
  // Ts_cat = s X [l1_0 | ... | l1_{G-1}]: one skinny GEMM for every member
  // (they share X), each member's columns stored as its [hi | lo] pair
  Operand A{x, K, 0}, B{l1, R, 1};
  rc = gemm::plain(64, A, B, m, R, K, s, ts_out, 2 * R, 0, 0, (float*)workspace, part_bytes, st, 0, rank, &sk);
  if (rc != QLRT_OK) return rc;
  // Y^T[N, m] = W_cat^T X^T + per member [l2_g ; l2_g]^T [Ts_g]^T
  gemm::Args a{};
  if ((rc = gemm::fill_nf4(a, w, 1, nullptr, st)) != QLRT_OK) return rc;
  a.M = (int)N;
  a.N = (int)m;
  a.splits = 1;
  a.out = y;
  a.ldo = N;
  a.out_t = 1;
  a.alpha = 1.0f;
  const int bn_main = gemm::tile512_policy() ? 512 : 256;
  a.pair = bn_main == 512 ? 1 : gemm::pair_policy(0);
  if (gemm::streamk_policy()) { a.sk_ws = sk.sk_ws; a.sk_flags = sk.sk_flags; }
  a.aug_wrap = rank;
  a.aug_gn = (int)Ng;
  a.aug_gstride = 2 * rank;
  a.aug_b2k = 2 * R;
  // the fused grid is the PDL dependent of Ts's split-K reduce: it starts its
  // main K loop as Ts's CTAs retire and waits for Ts_cat only before the
  // augmented segment (X, the only earlier input, is older than Ts)
  a.aug_pdl = gemm::pdl_policy() ? 1 : 0;
  Operand none{}, Bx{x, K, 0}, A2{l2, N, 1}, B2{ts_out, 2 * R, 0};
  return gemm::run(bn_main, none, Bx, &A2, &B2, K, 2 * rank, a, st);
}

qlrt_status qlrt_nf4_linear_group_bwd(const qlrt_nf4_weight* w, int groups, const void* dy, int64_t m,
                                      const void* x, const void* ts, const void* l1, const void* l2, int rank,
                                      float s, void* dt_out, void* dx, float* dl1, float* dl2, void* workspace,
                                      void* side_workspace, int flags, void* stream) {
  if (!group_ok(w, groups, rank) || !dy || !dx || !x || !ts || !l1 || !l2 || !dt_out || !dl1 || !dl2 ||
      !workspace || m <= 0 || (flags & ~QLRT_BWD_DEFER))
    return QLRT_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t K = w->k_in, N = w->n_out, Ng = N / groups;
  const int R = groups * rank;
  const size_t ws_bytes = qlrt_linear_workspace_bytes(m, K, N, R);
  const size_t part_bytes =
      ws_bytes - gemm::dbl_bytes(K, N, R) - gemm::sk_bytes() - gemm::align256(gemm::consts_bytes(K, N));
  gemm::Args sk{};
  gemm::sk_region(workspace, ws_bytes, K, N, R, sk);
  qlrt_status rc;
  typedef __nv_bfloat16 bf;
  // dT_g = s dY_g l2_g^T into member g's [hi | lo] block of dT_cat: one
  // grouped-K launch (column tile g reduces over member g's K range)
  {
    Operand DA{dy, N, 0}, DB{l2, N, 0};
    rc = gemm::plain(64, DA, DB, m, R, Ng, s, dt_out, 2 * R, 0, 0, (float*)workspace, part_bytes, st, 0, rank, &sk,
                     0, 0, 0, rank, N);
    if (rc != QLRT_OK) return rc;
  }
  gemm::SideCtx* sctx = gemm::side_ctx(st);
  const bool defer = (flags & QLRT_BWD_DEFER) && sctx && side_workspace;
  const int side_cap = defer ? policy(P_SIDE_SMS) : 0;
  cudaStream_t side = gemm::fork_side(sctx, st);
  // dX^T[K, m] = W_cat dY_cat^T + sum_g [l1_g | l1_g] [dT_g]^T (K2 = G 2r; the
  // wrapped A2 re-reads member g's l1 columns for both halves of its pair)
  gemm::Args a{};
  if ((rc = gemm::fill_nf4(a, w, 2, nullptr, st)) != QLRT_OK) return rc;
  a.M = (int)K;
  a.N = (int)m;
  a.splits = 1;
  a.out = dx;
  a.ldo = K;
  a.out_t = 1;
  a.alpha = 1.0f;
  const int bn_main = gemm::tile512_policy() ? 512 : 256;
  a.pair = bn_main == 512 ? 1 : gemm::pair_policy(0);
  if (gemm::streamk_policy()) { a.sk_ws = sk.sk_ws; a.sk_flags = sk.sk_flags; }
  a.aug_wrap = rank;
  Operand none{}, B{dy, N, 0}, A2{l1, R, 0}, B2{dt_out, 2 * R, 0};
  if ((rc = gemm::run(bn_main, none, B, &A2, &B2, N, 2 * R, a, st)) != QLRT_OK) return rc;
  cudaStream_t aux = side ? side : st;
  const int bn_g = 2 * rank <= 64 ? 64 : (2 * rank <= 128 ? 128 : 256);
  // dl2_g^T[N_g, r] = dY_g^T (Ts_g hi + lo), stored into columns g N_g.. of dl2[r][N]
  for (int g = 0; g < groups; ++g) {
    Operand A{(const bf*)dy + g * Ng, N, 1}, Bt{(const bf*)ts + 2 * g * rank, 2 * R, 1};
    rc = gemm::plain(bn_g, A, Bt, Ng, 2 * rank, m, 1.0f, dl2 + g * Ng, N, 1, 1, nullptr, 0, aux, rank, 0, nullptr, 0,
                     0, side_cap);
    if (rc != QLRT_OK) return rc;
  }
  {
    // dl1_cat[K, G r] = X^T (dT_cat hi + lo per member): one GEMM (the members share X)
    Operand A{x, K, 1}, B1{dt_out, 2 * R, 1};
    float* pw = defer ? (float*)side_workspace : (float*)workspace;
    rc = gemm::plain(2 * R <= 128 ? (2 * R <= 64 ? 64 : 128) : ((2 * R) % 256 == 0 ? 256 : 128), A, B1, K, 2 * R, m,
                     1.0f, dl1, R, 1, 0, pw,
                     part_bytes, aux, rank, 0, side ? nullptr : &sk, 0, 0, side_cap);
    if (rc != QLRT_OK) return rc;
  }
  if (side && !defer && !gemm::join_side(sctx, st)) return QLRT_ERR_CUDA;
  return QLRT_OK;
}

qlrt_status qlrt_nf4_linear_bwd(const qlrt_nf4_weight* w, const void* dy, int64_t m, const void* x, const void* ts,
                                const void* l1, const void* l2, int rank, float s, void* dt_out, void* dx, float* dl1,
                                float* dl2, void* workspace, void* stream) {
  return qlrt_nf4_linear_bwd_ex(w, dy, m, x, ts, l1, l2, rank, s, dt_out, dx, dl1, dl2, workspace, nullptr, 0,
                                stream);
}

void* qlrt_side_stream(void* stream) {
  gemm::SideCtx* c = policy(P_SIDE) ? gemm::side_ctx((cudaStream_t)stream) : nullptr;
  return c ? (void*)c->side : nullptr;
}

qlrt_status qlrt_side_join(void* stream) {
  // the caller's stream waits for everything issued on its side stream so far
  // (a no-op without one: nothing was deferred)
  if (!policy(P_SIDE)) return QLRT_OK;
  gemm::SideCtx* c = gemm::side_ctx((cudaStream_t)stream);
  if (!c) return QLRT_OK;
  return gemm::join_side(c, (cudaStream_t)stream) ? QLRT_OK : QLRT_ERR_CUDA;
}

}  // extern "C"
