// torch custom-op layer over the C ABI (include/qlrt_b200.h): the hot-path
// entry points as torch.ops.qlrt_b200.* schemas with a CUDA implementation
// (outputs from the caching allocator, launches on the current torch stream)
// and a Meta implementation (shapes / dtypes only, for fake tensors and
// tracing).  Each op mirrors a reference function (qlrt 0.1.0):
//   quantize4        blockquant.py:132-195 (phase A: codes + fp32 absmax)
//   dq_compress      doublequant.py:148-187
//   dequantize4      blockquant.py:198-213 (+ dq_decompress, doublequant.py:190-195)
//   nf4_linear_fwd   qlora.py:124-148  (QLinear.forward, one adapter, no dropout)
//   nf4_linear_bwd   qlora.py:150-167  (QLinear.backward)
//   nf4_gemv         qlora.py:124-148 at M = 1
//   adam_step        training.py:416-442 (in place)
// The Python mirror (paper_2305_14314_b200) binds the same C ABI with ctypes;
// this layer is for torch users (custom ops compose with autograd.Function,
// CUDA graphs, torch.compile).  Built by tools/build_lib.sh into
// _lib/libqlrt_torch_ops.so, linked against libqlrt_b200.so.
#include <ATen/ATen.h>
#include <ATen/cuda/CUDAContext.h>
#include <torch/library.h>

#include <cstring>

#include "qlrt_b200.h"

namespace {

using at::Tensor;

void ok(int st, const char* what) {
  TORCH_CHECK(st != QLRT_ERR_ARG, what, ": invalid argument");
  TORCH_CHECK(st == QLRT_OK, what, ": ", st == QLRT_ERR_CUDA ? "CUDA error" : "unsupported shape/layout");
}

void* stream() { return (void*)at::cuda::getCurrentCUDAStream().stream(); }

qlrt_codebook4 codebook_of(const Tensor& blob) {
  TORCH_CHECK(blob.device().is_cpu() && blob.scalar_type() == at::kByte &&
                  blob.numel() == (int64_t)sizeof(qlrt_codebook4),
              "codebook must be the qlrt_codebook4 struct as a CPU uint8 tensor (Codebook.to_c())");
  qlrt_codebook4 cb;
  std::memcpy(&cb, blob.contiguous().data_ptr(), sizeof cb);
  return cb;
}

qlrt_fp8spec spec_of(at::IntArrayRef s) {
  TORCH_CHECK(s.size() == 3, "fp8 spec is [exp_bits, mant_bits, bias]");
  return qlrt_fp8spec{(int)s[0], (int)s[1], (int)s[2]};
}

qlrt_nf4_weight weight_of(const Tensor& codes, const Tensor& dq_codes, const Tensor& c1, const Tensor& mu,
                          int64_t k_in, int64_t n_out, int64_t bs2, at::IntArrayRef spec, at::ArrayRef<double> values,
                          const Tensor* consts) {
  TORCH_CHECK(values.size() == 16, "values: the 16-entry decode table");
  for (const Tensor* t : {&codes, &dq_codes, &c1, &mu})
    TORCH_CHECK(t->is_cuda() && t->is_contiguous(), "weight tensors must be contiguous CUDA tensors");
  TORCH_CHECK(codes.numel() * 2 == k_in * n_out, "codes: k_in * n_out / 2 bytes");
  qlrt_nf4_weight w{};
  w.codes = codes.data_ptr<uint8_t>();
  w.dq_codes = dq_codes.data_ptr<uint8_t>();
  w.c1 = c1.data_ptr<float>();
  w.mu = mu.data_ptr<float>();
  w.k_in = k_in;
  w.n_out = n_out;
  w.blocksize2 = (int)bs2;
  w.spec = spec_of(spec);
  for (int i = 0; i < 16; ++i) w.values[i] = values[i];
  w.consts = consts ? consts->data_ptr<float>() : nullptr;
  return w;
}

int64_t rank_of(const c10::optional<Tensor>& l1) { return l1.has_value() ? l1->size(1) : 0; }

// A fresh zero-filled workspace (stream-K flags must start at 0).
Tensor workspace(const Tensor& like, int64_t m, int64_t k, int64_t n, int64_t r) {
  return at::zeros({(int64_t)qlrt_linear_workspace_bytes(m, k, n, (int)r)}, like.options().dtype(at::kByte));
}

// ---------------------------------------------------------------- CUDA
std::tuple<Tensor, Tensor, Tensor> quantize4_cuda(const Tensor& x, const Tensor& codebook, int64_t blocksize) {
  TORCH_CHECK(x.is_cuda(), "x must be a CUDA tensor");
  const auto xc = x.contiguous();
  const int dt = xc.scalar_type() == at::kFloat ? QLRT_F32 : xc.scalar_type() == at::kBFloat16 ? QLRT_BF16
                 : xc.scalar_type() == at::kDouble ? QLRT_F64 : -1;
  TORCH_CHECK(dt >= 0, "x must be float32, bfloat16 or float64");
  TORCH_CHECK(xc.numel() > 0, "cannot quantize an empty tensor");
  const qlrt_codebook4 cb = codebook_of(codebook);
  const int64_t n = xc.numel(), nb = (n + blocksize - 1) / blocksize;
  auto codes = at::empty({(nb * blocksize + 1) / 2}, xc.options().dtype(at::kByte));
  auto absmax = at::empty({nb}, xc.options().dtype(at::kFloat));
  auto bad = at::empty({1}, xc.options().dtype(at::kLong));
  ok(qlrt_quantize4(xc.data_ptr(), dt, n, (int)blocksize, &cb, codes.data_ptr<uint8_t>(), absmax.data_ptr<float>(),
                    bad.data_ptr<int64_t>(), stream()),
     "qlrt_b200::quantize4");
  return {codes, absmax, bad};
}

std::tuple<Tensor, Tensor, Tensor> dq_compress_cuda(const Tensor& absmax, int64_t bs2, at::IntArrayRef spec) {
  TORCH_CHECK(absmax.is_cuda() && absmax.scalar_type() == at::kFloat, "absmax: float32 CUDA tensor");
  const auto a = absmax.contiguous();
  const int64_t nb = a.numel();
  auto ws = at::zeros({(int64_t)qlrt_dq_workspace_bytes(nb)}, a.options().dtype(at::kByte));
  auto mu = at::empty({1}, a.options());
  auto c1 = at::empty({(nb + bs2 - 1) / bs2}, a.options());
  auto codes = at::empty({nb}, a.options().dtype(at::kByte));
  ok(qlrt_dq_compress(a.data_ptr<float>(), nb, (int)bs2, spec_of(spec), ws.data_ptr(), mu.data_ptr<float>(),
                      c1.data_ptr<float>(), codes.data_ptr<uint8_t>(), stream()),
     "qlrt_b200::dq_compress");
  return {mu, c1, codes};
}

Tensor dequantize4_cuda(const Tensor& codes, int64_t numel, int64_t blocksize, const Tensor& codebook,
                        const Tensor& dq_codes, const Tensor& c1, const Tensor& mu, int64_t bs2, at::IntArrayRef spec,
                        at::ScalarType dtype) {
  const int dt = dtype == at::kFloat ? QLRT_F32 : dtype == at::kBFloat16 ? QLRT_BF16 : dtype == at::kDouble ? QLRT_F64
                                                                                                            : -1;
  TORCH_CHECK(dt >= 0, "dtype must be float32, bfloat16 or float64");
  const qlrt_codebook4 cb = codebook_of(codebook);
  auto out = at::empty({numel}, codes.options().dtype(dtype));
  ok(qlrt_dequantize4(codes.data_ptr<uint8_t>(), numel, (int)blocksize, &cb, nullptr, dq_codes.data_ptr<uint8_t>(),
                      c1.data_ptr<float>(), mu.data_ptr<float>(), (int)bs2, spec_of(spec), out.data_ptr(), dt,
                      stream()),
     "qlrt_b200::dequantize4");
  return out;
}

std::tuple<Tensor, Tensor, Tensor> linear_fwd_cuda(const Tensor& x, const Tensor& codes, const Tensor& dq_codes,
                                                   const Tensor& c1, const Tensor& mu, int64_t k_in, int64_t n_out,
                                                   int64_t bs2, at::IntArrayRef spec, at::ArrayRef<double> values,
                                                   const c10::optional<Tensor>& l1, const c10::optional<Tensor>& l2,
                                                   double s) {
  TORCH_CHECK(x.is_cuda() && x.scalar_type() == at::kBFloat16 && x.dim() == 2 && x.size(1) == k_in,
              "x: bf16 CUDA [M, k_in]");
  const auto xc = x.contiguous();
  const int64_t m = xc.size(0), r = rank_of(l1);
  TORCH_CHECK(l1.has_value() == l2.has_value(), "l1 and l2 go together");
  auto consts = at::empty({(int64_t)qlrt_nf4_constants_bytes(k_in, n_out) / 4}, x.options().dtype(at::kFloat));
  qlrt_nf4_weight w = weight_of(codes, dq_codes, c1, mu, k_in, n_out, bs2, spec, values, &consts);
  ok(qlrt_nf4_constants(&w, consts.data_ptr<float>(), stream()), "qlrt_b200::nf4_linear_fwd(constants)");
  auto y = at::empty({m, n_out}, xc.options());
  auto ts = at::empty({m, 2 * r}, xc.options());
  auto ws = workspace(xc, m, k_in, n_out, r);
  Tensor l1c, l2c;
  if (r) {
    l1c = l1->contiguous();
    l2c = l2->contiguous();
    TORCH_CHECK(l1c.scalar_type() == at::kBFloat16 && l2c.scalar_type() == at::kBFloat16, "l1, l2: bf16");
  }
  ok(qlrt_nf4_linear_fwd(&w, xc.data_ptr(), nullptr, m, r ? l1c.data_ptr() : nullptr, r ? l2c.data_ptr() : nullptr,
                         (int)r, (float)s, r ? ts.data_ptr() : nullptr, y.data_ptr(), ws.data_ptr(), stream()),
     "qlrt_b200::nf4_linear_fwd");
  return {y, ts, consts};
}

std::tuple<Tensor, Tensor, Tensor> linear_bwd_cuda(const Tensor& dy, const Tensor& x, const Tensor& ts,
                                                   const Tensor& consts, const Tensor& codes, const Tensor& dq_codes,
                                                   const Tensor& c1, const Tensor& mu, int64_t k_in, int64_t n_out,
                                                   int64_t bs2, at::IntArrayRef spec, at::ArrayRef<double> values,
                                                   const c10::optional<Tensor>& l1, const c10::optional<Tensor>& l2,
                                                   double s) {
  TORCH_CHECK(dy.is_cuda() && dy.scalar_type() == at::kBFloat16 && dy.dim() == 2 && dy.size(1) == n_out,
              "dy: bf16 CUDA [M, n_out]");
  const auto dyc = dy.contiguous();
  const int64_t m = dyc.size(0), r = rank_of(l1);
  qlrt_nf4_weight w = weight_of(codes, dq_codes, c1, mu, k_in, n_out, bs2, spec, values, &consts);
  auto dx = at::empty({m, k_in}, dyc.options());
  auto dl1 = at::empty({k_in, r}, dyc.options().dtype(at::kFloat));
  auto dl2 = at::empty({r, n_out}, dyc.options().dtype(at::kFloat));
  auto dt = at::empty({m, 2 * r}, dyc.options());
  auto ws = workspace(dyc, m, k_in, n_out, r);
  Tensor xc, tsc, l1c, l2c;
  if (r) {
    xc = x.contiguous();
    tsc = ts.contiguous();
    l1c = l1->contiguous();
    l2c = l2->contiguous();
  }
  ok(qlrt_nf4_linear_bwd(&w, dyc.data_ptr(), m, r ? xc.data_ptr() : nullptr, r ? tsc.data_ptr() : nullptr,
                         r ? l1c.data_ptr() : nullptr, r ? l2c.data_ptr() : nullptr, (int)r, (float)s,
                         r ? dt.data_ptr() : nullptr, dx.data_ptr(), r ? dl1.data_ptr<float>() : nullptr,
                         r ? dl2.data_ptr<float>() : nullptr, ws.data_ptr(), stream()),
     "qlrt_b200::nf4_linear_bwd");
  return {dx, dl1, dl2};
}

Tensor gemv_cuda(const Tensor& x, const Tensor& codes, const Tensor& dq_codes, const Tensor& c1, const Tensor& mu,
                 int64_t k_in, int64_t n_out, int64_t bs2, at::IntArrayRef spec, at::ArrayRef<double> values,
                 const c10::optional<Tensor>& l1, const c10::optional<Tensor>& l2, double s) {
  TORCH_CHECK(x.is_cuda() && x.scalar_type() == at::kBFloat16 && x.numel() == k_in, "x: bf16 CUDA [1, k_in]");
  const auto xc = x.contiguous();
  const int64_t r = rank_of(l1);
  qlrt_nf4_weight w = weight_of(codes, dq_codes, c1, mu, k_in, n_out, bs2, spec, values, nullptr);
  auto y = at::empty({1, n_out}, xc.options());
  auto ws = workspace(xc, 1, k_in, n_out, r);
  Tensor l1c, l2c;
  if (r) {
    l1c = l1->contiguous();
    l2c = l2->contiguous();
  }
  ok(qlrt_nf4_gemv(&w, xc.data_ptr(), nullptr, r ? l1c.data_ptr() : nullptr, r ? l2c.data_ptr() : nullptr, (int)r,
                   (float)s, y.data_ptr(), ws.data_ptr(), stream()),
     "qlrt_b200::nf4_gemv");
  return y;
}

void adam_cuda(Tensor& p, const Tensor& g, Tensor& m, Tensor& v, double b1, double omb1, double b2, double omb2,
               double bc1, double bc2, double eps, double lr) {
  for (const Tensor* t : {(const Tensor*)&p, &g, (const Tensor*)&m, (const Tensor*)&v})
    TORCH_CHECK(t->is_cuda() && t->is_contiguous() && t->scalar_type() == at::kFloat && t->numel() == p.numel(),
                "adam_step: contiguous float32 CUDA tensors of one size");
  ok(qlrt_adam_step(p.data_ptr<float>(), g.data_ptr<float>(), m.data_ptr<float>(), v.data_ptr<float>(), p.numel(),
                    (float)b1, (float)omb1, (float)b2, (float)omb2, (float)bc1, (float)bc2, (float)eps, (float)lr,
                    nullptr, stream()),
     "qlrt_b200::adam_step");
}

// ---------------------------------------------------------------- Meta
std::tuple<Tensor, Tensor, Tensor> quantize4_meta(const Tensor& x, const Tensor&, int64_t blocksize) {
  const int64_t nb = (x.numel() + blocksize - 1) / blocksize;
  return {at::empty({(nb * blocksize + 1) / 2}, x.options().dtype(at::kByte)),
          at::empty({nb}, x.options().dtype(at::kFloat)), at::empty({1}, x.options().dtype(at::kLong))};
}

std::tuple<Tensor, Tensor, Tensor> dq_compress_meta(const Tensor& a, int64_t bs2, at::IntArrayRef) {
  return {at::empty({1}, a.options()), at::empty({(a.numel() + bs2 - 1) / bs2}, a.options()),
          at::empty({a.numel()}, a.options().dtype(at::kByte))};
}

Tensor dequantize4_meta(const Tensor& codes, int64_t numel, int64_t, const Tensor&, const Tensor&, const Tensor&,
                        const Tensor&, int64_t, at::IntArrayRef, at::ScalarType dtype) {
  return at::empty({numel}, codes.options().dtype(dtype));
}

std::tuple<Tensor, Tensor, Tensor> linear_fwd_meta(const Tensor& x, const Tensor&, const Tensor&, const Tensor&,
                                                   const Tensor&, int64_t k_in, int64_t n_out, int64_t, at::IntArrayRef,
                                                   at::ArrayRef<double>, const c10::optional<Tensor>& l1,
                                                   const c10::optional<Tensor>&, double) {
  const int64_t m = x.size(0), r = rank_of(l1);
  return {at::empty({m, n_out}, x.options()), at::empty({m, 2 * r}, x.options()),
          at::empty({(int64_t)qlrt_nf4_constants_bytes(k_in, n_out) / 4}, x.options().dtype(at::kFloat))};
}

std::tuple<Tensor, Tensor, Tensor> linear_bwd_meta(const Tensor& dy, const Tensor&, const Tensor&, const Tensor&,
                                                   const Tensor&, const Tensor&, const Tensor&, const Tensor&,
                                                   int64_t k_in, int64_t n_out, int64_t, at::IntArrayRef,
                                                   at::ArrayRef<double>, const c10::optional<Tensor>& l1,
                                                   const c10::optional<Tensor>&, double) {
  const int64_t m = dy.size(0), r = rank_of(l1);
  return {at::empty({m, k_in}, dy.options()), at::empty({k_in, r}, dy.options().dtype(at::kFloat)),
          at::empty({r, n_out}, dy.options().dtype(at::kFloat))};
}

Tensor gemv_meta(const Tensor& x, const Tensor&, const Tensor&, const Tensor&, const Tensor&, int64_t, int64_t n_out,
                 int64_t, at::IntArrayRef, at::ArrayRef<double>, const c10::optional<Tensor>&,
                 const c10::optional<Tensor>&, double) {
  return at::empty({1, n_out}, x.options());
}

void adam_meta(Tensor&, const Tensor&, Tensor&, Tensor&, double, double, double, double, double, double, double,
               double) {}

}  // namespace

TORCH_LIBRARY(qlrt_b200, m) {
  m.def("quantize4(Tensor x, Tensor codebook, int blocksize) -> (Tensor codes, Tensor absmax, Tensor first_bad)");
  m.def("dq_compress(Tensor absmax, int blocksize2, int[3] spec) -> (Tensor mu, Tensor c1, Tensor codes)");
  m.def("dequantize4(Tensor codes, int numel, int blocksize, Tensor codebook, Tensor dq_codes, Tensor c1, Tensor mu, "
        "int blocksize2, int[3] spec, ScalarType dtype) -> Tensor");
  m.def("nf4_linear_fwd(Tensor x, Tensor codes, Tensor dq_codes, Tensor c1, Tensor mu, int k_in, int n_out, "
        "int blocksize2, int[3] spec, float[] values, Tensor? l1, Tensor? l2, float s) -> (Tensor y, Tensor ts, "
        "Tensor consts)");
  m.def("nf4_linear_bwd(Tensor dy, Tensor x, Tensor ts, Tensor consts, Tensor codes, Tensor dq_codes, Tensor c1, "
        "Tensor mu, int k_in, int n_out, int blocksize2, int[3] spec, float[] values, Tensor? l1, Tensor? l2, "
        "float s) -> (Tensor dx, Tensor dl1, Tensor dl2)");
  m.def("nf4_gemv(Tensor x, Tensor codes, Tensor dq_codes, Tensor c1, Tensor mu, int k_in, int n_out, "
        "int blocksize2, int[3] spec, float[] values, Tensor? l1, Tensor? l2, float s) -> Tensor");
  m.def("adam_step(Tensor(a!) p, Tensor g, Tensor(b!) m, Tensor(c!) v, float b1, float omb1, float b2, float omb2, "
        "float bc1, float bc2, float eps, float lr) -> ()");
}

TORCH_LIBRARY_IMPL(qlrt_b200, CUDA, m) {
  m.impl("quantize4", &quantize4_cuda);
  m.impl("dq_compress", &dq_compress_cuda);
  m.impl("dequantize4", &dequantize4_cuda);
  m.impl("nf4_linear_fwd", &linear_fwd_cuda);
  m.impl("nf4_linear_bwd", &linear_bwd_cuda);
  m.impl("nf4_gemv", &gemv_cuda);
  m.impl("adam_step", &adam_cuda);
}

TORCH_LIBRARY_IMPL(qlrt_b200, Meta, m) {
  m.impl("quantize4", &quantize4_meta);
  m.impl("dq_compress", &dq_compress_meta);
  m.impl("dequantize4", &dequantize4_meta);
  m.impl("nf4_linear_fwd", &linear_fwd_meta);
  m.impl("nf4_linear_bwd", &linear_bwd_meta);
  m.impl("nf4_gemv", &gemv_meta);
  m.impl("adam_step", &adam_meta);
}
