/*
 * qlrt_b200.h -- C ABI of the B200-native NF4 / double-quant / QLoRA-linear
 * hot path.  Every entry point takes DEVICE pointers, element counts and a
 * cudaStream_t (passed as void*), never allocates (callers own all buffers,
 * including the documented workspaces) and returns a qlrt_status.  Launches
 * are stream-ordered and reentrant.  Process-wide state is limited to the
 * launch-policy table (atomics, qlrt_set_policy) and a mutex-guarded table of
 * side streams keyed by (device, caller stream), so callers on different
 * streams never share a side stream or its fork/join events.
 *
 * Each function cites the reference (qlrt 0.1.0, /root/reference/pkg/src/qlrt)
 * interface it replaces.  The Python host mirror binds these with ctypes
 * (paper_2305_14314_b200/_native.py); INTEGRATION.md shows the binding.
 */
#ifndef QLRT_B200_H
#define QLRT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QLRT_OK = 0,
  QLRT_ERR_ARG = 1,        /* ValueError in the reference                         */
  QLRT_ERR_CUDA = 2,       /* launch / runtime failure                            */
  QLRT_ERR_UNSUPPORTED = 3 /* shape/layout outside what the kernel was built for  */
} qlrt_status;

typedef enum { QLRT_F32 = 0, QLRT_BF16 = 1, QLRT_F64 = 2 } qlrt_dtype;

/* A 4-bit codebook as the kernels consume it (codebooks.py:125-176).
 * values: the 16-entry decode table (spares duplicate 0.0);
 * mids: the n_mids = n_emitted-1 fp64 decision boundaries;
 * lo/hi: fp32 brackets around each midpoint -- outside [lo,hi] the fp32 fast
 * path decides the code, inside it the kernel re-decides in fp64;
 * pad_code: code of padding and of all-zero blocks (blockquant.py:173-179). */
typedef struct {
  double values[16];
  double mids[15];
  float lo[16];
  float hi[16];
  int n_mids;
  int pad_code;
} qlrt_codebook4;

/* 8-bit float layout of the double quantizer (doublequant.py:33-51). */
typedef struct {
  int exp_bits;
  int mant_bits;
  int bias;
} qlrt_fp8spec;

/* ---- quantization (blockquant.py:132-195, doublequant.py:148-187) ------- */

/* Phase A of quantize(): per-block float32 absmax, nearest codes (ties away
 * from zero, fp64-exact), 2-codes-per-byte packing, padding/zero blocks ->
 * pad_code, first non-finite flat index (>= n if none: 0x7F7F7F7F7F7F7F7F).
 * x: n elements of x_dtype (F32, BF16 or F64 -- the reference's own dtype).  codes: ceil(nb*blocksize/2) bytes.
 * absmax: nb floats.  first_bad: one int64 on the device. */
qlrt_status qlrt_quantize4(const void* x, int x_dtype, int64_t n, int blocksize,
                           const qlrt_codebook4* cb, uint8_t* codes, float* absmax,
                           int64_t* first_bad, void* stream);

/* Bytes of scratch qlrt_dq_compress needs for nb constants. */
size_t qlrt_dq_workspace_bytes(int64_t nb);

/* dq_compress(): mu = f32(numpy-order mean), per-blocksize2 fp64 absmax,
 * c1 = f32(A/max), codes = nearest 8-bit float (ties away, clamp). */
qlrt_status qlrt_dq_compress(const float* absmax, int64_t nb, int blocksize2,
                             qlrt_fp8spec spec, void* workspace, float* mu, float* c1,
                             uint8_t* dq_codes, void* stream);

/* dq_decompress() (doublequant.py:190-195): nb float32 constants. */
qlrt_status qlrt_dq_decompress(const uint8_t* dq_codes, const float* c1, const float* mu,
                               int64_t nb, int blocksize2, qlrt_fp8spec spec, float* out,
                               void* stream);

/* dequantize() (blockquant.py:198-213): out[i] = f32(values[code_i] * f64(c_b)),
 * written as F64 (the reference's float64, bit-exact), F32 or BF16 (bf16 of the f32).  Either absmax (plain constants)
 * or (dq_codes, c1, mu) must be given (4-bit codes cannot leave the table). */
qlrt_status qlrt_dequantize4(const uint8_t* codes, int64_t n, int blocksize,
                             const qlrt_codebook4* cb, const float* absmax,
                             const uint8_t* dq_codes, const float* c1, const float* mu,
                             int blocksize2, qlrt_fp8spec spec, void* out, int out_dtype,
                             void* stream);

/* encode_fp8 / decode_fp8 (doublequant.py:103-121) on arbitrary fp64 values. */
qlrt_status qlrt_fp8_encode(const double* x, int64_t n, qlrt_fp8spec spec, uint8_t* out, void* stream);
qlrt_status qlrt_fp8_decode(const uint8_t* codes, int64_t n, qlrt_fp8spec spec, double* out, void* stream);

/* pack_codes / unpack_codes (blockquant.py:81-115) for k = 4. */
qlrt_status qlrt_pack4(const uint8_t* codes, int64_t count, uint8_t* packed, void* stream);
qlrt_status qlrt_unpack4(const uint8_t* packed, int64_t count, uint8_t* codes, void* stream);

/* ---- frozen NF4 linear with LoRA (qlora.py:117-167) ---------------------- */

/* The quantized base W[K_in, N_out] (row-major, blocks of 64 along N_out,
 * qlora.py:110-115) in the form the fused kernels read. */
typedef struct {
  const uint8_t* codes;    /* K_in*N_out/2 bytes                         */
  const uint8_t* dq_codes; /* K_in*N_out/64 bytes                        */
  const float* c1;         /* ceil(nb/blocksize2) floats                 */
  const float* mu;         /* 1 float (device)                           */
  int64_t k_in, n_out;
  int blocksize2;
  qlrt_fp8spec spec;
  double values[16];       /* codebook decode table                      */
  float* consts;           /* optional fp32 block-constant cache [k_in][round4(n_out/64)]:
                              NULL -> rebuilt in the workspace every call;
                              non-NULL -> (re)built by qlrt_nf4_constants,
                              read by fwd/bwd/gemv (the reference caches the
                              dequantized W from forward to backward,
                              qlora.py:146-147,179) */
} qlrt_nf4_weight;

/* Bytes of the constant cache of a weight and the call that fills it
 * (doublequant.py:190-195 arithmetic, laid out for the fused GEMM). */
size_t qlrt_nf4_constants_bytes(int64_t k_in, int64_t n_out);
qlrt_status qlrt_nf4_constants(const qlrt_nf4_weight* w, float* out, void* stream);

/* One weight's block constants into columns [0, n_out/64) of rows of `pitch`
 * floats: a member's slice of a concatenated (grouped) weight's cache. */
qlrt_status qlrt_nf4_constants_into(const qlrt_nf4_weight* w, float* out, int64_t pitch, void* stream);
/* The same for up to 4 sibling weights of one shape in one launch (member g
 * in columns [g n_out/64, (g + 1) n_out/64)). */
qlrt_status qlrt_nf4_constants_group(const qlrt_nf4_weight* members, int groups, float* out, int64_t pitch,
                                     void* stream);

/* Step-level prepass: the block constants of many weights in one launch.
 * jobs_dev (device memory) lists, per weight (or member of a group), its DQ
 * data and where its [rows][nbr] constants go (row pitch `pitch` floats);
 * max_elems = the largest rows * nbr.  The fused kernels then read the
 * caches (qlrt_nf4_weight.consts) instead of rebuilding them per call. */
typedef struct {
  const uint8_t* dq_codes;
  const float* c1;
  const float* mu;
  float* out;
  int64_t rows, nbr, pitch;
  int blocksize2;
  qlrt_fp8spec spec;
} qlrt_nf4_const_job;
qlrt_status qlrt_nf4_constants_batch(const qlrt_nf4_const_job* jobs_dev, int n_jobs, int64_t max_elems,
                                     void* stream);

/* Workspace bytes for the linear entry points (split-K partial sums). */
/* (The workspace also holds the stream-K partial tiles and flags: the caller
 * zero-fills a new workspace once -- the flags must start at 0, and every
 * launch leaves them 0 again.) */
size_t qlrt_linear_workspace_bytes(int64_t m, int64_t k_in, int64_t n_out, int rank);

/* forward (qlora.py:124-148):
 *   Ts = s * Xa l1 as a bf16 hi/lo pair [M, 2r] (Ts[:, :r] + Ts[:, r:]; kept for backward)
 *   Y  = X W + (Ts_hi + Ts_lo) l2       [M, N]   bf16 out, fp32 accumulate
 *        (one augmented K = 2r segment of the same tcgen05 accumulator)
 * X bf16 [M,K]; Xa = the adapter input (X with the dropout mask applied,
 * qlora.py:137-143; NULL -> X); l1 bf16 [K,r], l2 bf16 [r,N]; rank % 8 == 0
 * (callers zero-pad), rank == 0 -> no adapter.  N % 64 == 0, K % 8 == 0. */
qlrt_status qlrt_nf4_linear_fwd(const qlrt_nf4_weight* w, const void* x, const void* xa,
                                int64_t m, const void* l1, const void* l2, int rank, float s,
                                void* ts_out, void* y, void* workspace, void* stream);

/* backward (qlora.py:150-167):
 *   dT  = s * dY l2^T as a bf16 hi/lo pair [M, 2r]
 *   dX  = dY W^T + (dT_hi + dT_lo) l1^T [M, K]  bf16
 *   dl2 = (Ts_hi + Ts_lo)^T dY          [r, N]  fp32   (= s T^T dY)
 *   dl1 = Xa^T (dT_hi + dT_lo)          [K, r]  fp32   (= s Xa^T dY l2^T)
 * The hi/lo pairs keep the adapter gradients at ~16-bit operand precision.
 * (x is the adapter input Xa; with dropout the caller masks the adapter part
 * of dX itself and passes rank = 0 semantics through qlrt_gemm_bf16.) */
qlrt_status qlrt_nf4_linear_bwd(const qlrt_nf4_weight* w, const void* dy, int64_t m,
                                const void* x, const void* ts, const void* l1,
                                const void* l2, int rank, float s, void* dt_out, void* dx,
                                float* dl1, float* dl2, void* workspace, void* stream);

/* backward with flags.  QLRT_BWD_DEFER: the adapter-gradient GEMMs (dl2, dl1)
 * are left on the library's side stream of `stream` and NOT joined: they run
 * beside whatever the caller issues next (the following layers' fused grids
 * leave SMs idle) until qlrt_side_join(stream).  The caller must then keep x,
 * ts, dy and dt_out alive and unmodified, and not read dl1 / dl2, until it has
 * issued qlrt_side_join; side_workspace (>= qlrt_linear_workspace_bytes of
 * the call, distinct from `workspace`) holds the deferred split-K partials.
 * flags = 0 is qlrt_nf4_linear_bwd.  (The reference computes the gradients in
 * the same call, qlora.py:150-167; only their completion point moves.) */
#define QLRT_BWD_DEFER 1
qlrt_status qlrt_nf4_linear_bwd_ex(const qlrt_nf4_weight* w, const void* dy, int64_t m,
                                   const void* x, const void* ts, const void* l1,
                                   const void* l2, int rank, float s, void* dt_out, void* dx,
                                   float* dl1, float* dl2, void* workspace,
                                   void* side_workspace, int flags, void* stream);
/* `stream` waits for everything deferred on its side stream so far. */
qlrt_status qlrt_side_join(void* stream);
/* The side stream of `stream` (cudaStream_t; NULL when side streams are off),
 * for callers that order against part of the deferred work with their own
 * events. */
void* qlrt_side_stream(void* stream);

/* Sibling projections that share their input (q | k | v, gate | up) as one
 * call: w describes W_cat = [W_0 | ... | W_{groups-1}] (codes concatenated
 * along N, n_out = groups N_g, N_g % 256 == 0; every member quantized on
 * its own -- the reference's per-layer QLinear -- its constants placed by
 * qlrt_nf4_constants_into into w->consts, which is required); one adapter
 * of rank r (r % 64 == 0) per member, l1_cat [K][groups r], l2_cat
 * [r][n_out] bf16.  Ts_cat / dT_cat [M][groups 2r] hold each member's bf16
 * [hi | lo] pair; Y, dY [M][n_out]; dl1 [K][groups r], dl2 [r][n_out] fp32.
 * Same math per member as qlrt_nf4_linear_fwd / _bwd_ex (qlora.py:124-167):
 * Ts for all members is one GEMM, the fused NF4 GEMM covers every member
 * (the backward sums dX over them in its accumulator), dl1 is one GEMM. */
qlrt_status qlrt_nf4_linear_group_fwd(const qlrt_nf4_weight* w, int groups, const void* x,
                                      int64_t m, const void* l1, const void* l2, int rank,
                                      float s, void* ts_out, void* y, void* workspace,
                                      void* stream);
qlrt_status qlrt_nf4_linear_group_bwd(const qlrt_nf4_weight* w, int groups, const void* dy,
                                      int64_t m, const void* x, const void* ts, const void* l1,
                                      const void* l2, int rank, float s, void* dt_out, void* dx,
                                      float* dl1, float* dl2, void* workspace,
                                      void* side_workspace, int flags, void* stream);

/* batch-1 GEMV variant of forward (M = 1), HBM-bound on the packed codes:
 *   y[N] = x[K] W + s (xa l1) l2         fp32 accumulate, bf16 out
 * (xa = the dropout-masked adapter input, NULL -> x; qlora.py:137-146).
 * N % 256 == 0, K % 32 == 0 (the LLaMA shapes): tensor-core GEMV, W enters
 * as fp16(v) * c (the reference's float32 W to ~2^-12); other shapes: W
 * decodes as bf16(f32(v) * c) (as the fused GEMM).  Split-K partials are
 * summed in a fixed order (deterministic).  Needs N % 64 == 0, a
 * power-of-two blocksize2, 32-byte aligned codes; rank <= 512. */
qlrt_status qlrt_nf4_gemv(const qlrt_nf4_weight* w, const void* x, const void* xa,
                          const void* l1, const void* l2, int rank, float s, void* y,
                          void* workspace, void* stream);

/* Workspace bytes of qlrt_nf4_gemv (split-K partials, LoRA partials, strip
 * tickets); qlrt_linear_workspace_bytes(m = 1, ...) already covers it. */
size_t qlrt_gemv_workspace_bytes(int64_t k_in, int64_t n_out, int rank);

/* Plain bf16 GEMM on the same tcgen05 engine (test + building block):
 * D[M,N] = alpha * A[M,K] B[K,N]; a_mn/b_mn select MN-major storage
 * (A stored [K,M] / B stored [K,N]) vs K-major (A [M,K] / B [N,K]).
 * out_f32 selects fp32 vs bf16 output, out_t stores D^T ([N,M]).  A workspace
 * of >= ~19.5 MB reserves its tail for stream-K (zero-filled once, as above). */
qlrt_status qlrt_gemm_bf16(const void* a, const void* b, void* d, int64_t m, int64_t n,
                           int64_t k, int a_mn, int b_mn, float alpha, int out_f32,
                           int out_t, void* workspace, size_t workspace_bytes,
                           void* stream);

/* ---- optimizer (training.py:398-442) ------------------------------------ */

/* Bit-exact fp32 Adam (training.py:434-440 op order); also refreshes the
 * bf16 shadow copy used by the GEMMs when p_bf16 != NULL.  The constants are
 * the float32-rounded values numpy 2 uses (b1, 1-b1, b2, 1-b2, bc1, bc2,
 * eps, lr). */
qlrt_status qlrt_adam_step(float* p, const float* g, float* m, float* v, int64_t n,
                           float b1, float omb1, float b2, float omb2, float bc1,
                           float bc2, float eps, float lr, void* p_bf16, void* stream);

/* The same update over one flat buffer with its scalars in device memory
 * (hyper[8] = b1, 1-b1, b2, 1-b2, bc1, bc2, eps, lr: a CUDA graph replays it
 * while the host refreshes hyper) and, when sumsq != NULL, the global-norm
 * clip fused in: g *= f32(max_norm / sqrt(*sumsq)) if that norm > max_norm
 * (training.py:398-413).  16-byte aligned p, g, m, v; 8-byte aligned p_bf16. */
qlrt_status qlrt_adam_step_dev(float* p, const float* g, float* m, float* v, int64_t n,
                               const float* hyper, const double* sumsq, double max_norm,
                               void* p_bf16, void* stream);

/* sum of squares in fp64 of n floats (4-byte aligned), accumulated into acc[0] (device).
 * acc must have QLRT_SUMSQ_SCRATCH bytes: acc[0] result, then scratch. */
#define QLRT_SUMSQ_SCRATCH (8 + 8 * 296 + 8)
qlrt_status qlrt_sumsq_f64(const float* g, int64_t n, double* acc, void* stream);

/* g *= scale (float32), for clip_global_norm. */
/* clip_global_norm's per-tensor sum in numpy's own order: acc +=
 * pairwise_sum(float64(g)^2) (np.sum(np.square(g, dtype=float64)),
 * loops_utils.h.src).  The tree depends on n only and is built by the caller:
 * leaves [n_leaves][2] = (offset, length <= 128) in order, internal nodes
 * ops [][3] = (dst, left, right) indices into vals (leaves first), grouped
 * by height (level_starts[n_levels + 1]), root = the index of the sum;
 * vals >= n_leaves + #ops doubles. */
qlrt_status qlrt_sumsq_f64_pairwise(const float* g, const int* leaves, int n_leaves, const int* ops,
                                    const int* level_starts, int n_levels, int root, double* vals, double* acc,
                                    void* stream);
qlrt_status qlrt_scale_f32(float* g, int64_t n, float scale, void* stream);

/* Paged optimizer state: advise + prefetch a managed range to a device
 * (device >= 0) or to the host (device < 0) on the given stream. */
qlrt_status qlrt_prefetch(void* ptr, size_t bytes, int device, void* stream);

/* ---- fused glue of the LLaMA-shaped harness (llama.py; not a reference path) */
/* bf16 in/out, fp32 math, 16-byte vectors (widths multiples of 8). */
qlrt_status qlrt_rmsnorm_fwd(const void* x, void* y, float* rstd, int64_t rows, int64_t h,
                             float eps, void* stream);
qlrt_status qlrt_rmsnorm_bwd(const void* dy, const void* x, const float* rstd, void* dx,
                             int64_t rows, int64_t h, void* stream);
/* The residual add fused into the next norm: s = bf16(x + d), y = rmsnorm(s);
 * and the norm's backward plus the residual branch: dx = rmsnorm_bwd(dy) + dres. */
qlrt_status qlrt_add_rmsnorm_fwd(const void* x, const void* d, void* s, void* y, float* rstd, int64_t rows,
                                 int64_t h, float eps, void* stream);
qlrt_status qlrt_rmsnorm_bwd_add(const void* dy, const void* x, const float* rstd, const void* dres, void* dx,
                                 int64_t rows, int64_t h, void* stream);
qlrt_status qlrt_swiglu_fwd(const void* g, const void* u, void* out, int64_t n, void* stream);
qlrt_status qlrt_swiglu_bwd(const void* g, const void* u, const void* dout, void* dg, void* du,
                            int64_t n, void* stream);
/* rotary embedding on [rows = b*s][heads][d], adjacent pairs; cos_sin fp32
 * [seq][d/2] (cos, sin); inverse = 1 rotates back (the backward). */
qlrt_status qlrt_rope(const void* x, void* y, const void* cos_sin, int64_t rows, int heads, int d,
                      int seq, int inverse, void* stream);
/* RoPE with row pitches (elements): q / k read from or written to a column
 * slice of the concatenated q | k | v projection. */
qlrt_status qlrt_rope_strided(const void* x, int64_t ldx, void* y, int64_t ldy, const void* cos_sin,
                              int64_t rows, int heads, int d, int seq, int inverse, void* stream);
/* q | k | v rows of the concatenated projection -> rotated q, k and a copy
 * of v ([rows][heads d] each); backward: inverse-rotated dq, dk and dv into
 * the concatenated d[q | k | v] rows (one pass each way). */
qlrt_status qlrt_rope_qkv_fwd(const void* ycat, void* q, void* k, void* v, const void* cos_sin, int64_t rows,
                              int heads, int d, int seq, void* stream);
qlrt_status qlrt_rope_qkv_bwd(const void* dq, const void* dk, const void* dv, void* dycat, const void* cos_sin,
                              int64_t rows, int heads, int d, int seq, void* stream);
/* Cross entropy of bf16 logit rows (targets in [0, vocab)): per-row loss =
 * logsumexp - logit[target] and the row's logsumexp (fp32); backward writes
 * bf16 d logits = (softmax - onehot) * grad / rows (mean reduction; grad =
 * the device scalar upstream gradient). */
qlrt_status qlrt_xent_fwd(const void* logits, const int64_t* targets, int64_t rows, int64_t vocab, float* loss,
                          float* lse, void* stream);
qlrt_status qlrt_xent_bwd(const void* logits, const int64_t* targets, const float* lse, const float* grad,
                          int64_t rows, int64_t vocab, void* dlogits, void* stream);
/* SwiGLU over a concatenated [gate | up] projection (rows x 2 cols): out =
 * silu(g) * u [rows][cols]; backward writes d[gate | up]. */
qlrt_status qlrt_swiglu_cat_fwd(const void* gu, void* out, int64_t rows, int64_t cols, void* stream);
qlrt_status qlrt_swiglu_cat_bwd(const void* gu, const void* dout, void* dgu, int64_t rows, int64_t cols,
                                void* stream);

/* Launch-policy switches of the engine (the measured A/B knobs DESIGN.md
 * lists: QLRT_PAIR, QLRT_STREAMK, QLRT_OVERLAP, QLRT_OVERLAP_BWD, ...).  They
 * are read from the environment once, on first use; afterwards these calls
 * are the only way to change them (process-wide, atomic; no getenv on the
 * launch path).  value = INT32_MIN + 1 restores the built-in default.
 * Returns QLRT_ERR_ARG for an unknown name. */
int qlrt_set_policy(const char* name, int value);
int qlrt_get_policy(const char* name, int* value);

/* Library identification: returns the compiled arch string ("sm_100a"). */
const char* qlrt_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* QLRT_B200_H */
