"""ctypes binding of the C ABI in ``include/qlrt_b200.h``.

The CUDA library ``_lib/libqlrt_b200.so`` is built in-tree for sm_100a by
``tools/build_lib.sh`` (``__graft_entry__.build()``).  There is no CPU
fallback: every product entry point goes through this module and raises
``RuntimeError`` when the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int64, c_size_t, c_uint8, c_void_p

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QLRT_LIB_PATH") or os.path.join(_HERE, "_lib", "libqlrt_b200.so")

QLRT_OK, QLRT_ERR_ARG, QLRT_ERR_CUDA, QLRT_ERR_UNSUPPORTED = 0, 1, 2, 3
QLRT_BWD_DEFER = 1
F32, BF16, F64 = 0, 1, 2
SUMSQ_SCRATCH = 8 + 8 * 296 + 8


class Codebook4(ctypes.Structure):
    _fields_ = [("values", c_double * 16), ("mids", c_double * 15), ("lo", c_float * 16),
                ("hi", c_float * 16), ("n_mids", c_int), ("pad_code", c_int)]


class Fp8SpecC(ctypes.Structure):
    _fields_ = [("exp_bits", c_int), ("mant_bits", c_int), ("bias", c_int)]


class NF4Weight(ctypes.Structure):
    _fields_ = [("codes", c_void_p), ("dq_codes", c_void_p), ("c1", c_void_p), ("mu", c_void_p),
                ("k_in", c_int64), ("n_out", c_int64), ("blocksize2", c_int),
                ("spec", Fp8SpecC), ("values", c_double * 16), ("consts", c_void_p)]


class ConstJob(ctypes.Structure):
    _fields_ = [("dq_codes", c_void_p), ("c1", c_void_p), ("mu", c_void_p), ("out", c_void_p), ("rows", c_int64),
                ("nbr", c_int64), ("pitch", c_int64), ("blocksize2", c_int), ("spec", Fp8SpecC)]


_SIGS = {
    "qlrt_quantize4": [c_void_p, c_int, c_int64, c_int, POINTER(Codebook4), c_void_p, c_void_p, c_void_p, c_void_p],
    "qlrt_dq_workspace_bytes": [c_int64],
    "qlrt_dq_compress": [c_void_p, c_int64, c_int, Fp8SpecC, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "qlrt_dq_decompress": [c_void_p, c_void_p, c_void_p, c_int64, c_int, Fp8SpecC, c_void_p, c_void_p],
    "qlrt_dequantize4": [c_void_p, c_int64, c_int, POINTER(Codebook4), c_void_p, c_void_p, c_void_p, c_void_p,
                         c_int, Fp8SpecC, c_void_p, c_int, c_void_p],
    "qlrt_fp8_encode": [c_void_p, c_int64, Fp8SpecC, c_void_p, c_void_p],
    "qlrt_fp8_decode": [c_void_p, c_int64, Fp8SpecC, c_void_p, c_void_p],
    "qlrt_pack4": [c_void_p, c_int64, c_void_p, c_void_p],
    "qlrt_unpack4": [c_void_p, c_int64, c_void_p, c_void_p],
    "qlrt_linear_workspace_bytes": [c_int64, c_int64, c_int64, c_int],
    "qlrt_nf4_constants_bytes": [c_int64, c_int64],
    "qlrt_nf4_constants": [POINTER(NF4Weight), c_void_p, c_void_p],
    "qlrt_nf4_linear_fwd": [POINTER(NF4Weight), c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int, c_float,
                            c_void_p, c_void_p, c_void_p, c_void_p],
    "qlrt_nf4_linear_bwd": [POINTER(NF4Weight), c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                            c_float, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "qlrt_nf4_linear_bwd_ex": [POINTER(NF4Weight), c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                               c_float, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p],
    "qlrt_nf4_constants_into": [POINTER(NF4Weight), c_void_p, c_int64, c_void_p],
    "qlrt_nf4_constants_group": [POINTER(NF4Weight), c_int, c_void_p, c_int64, c_void_p],
    "qlrt_nf4_constants_batch": [c_void_p, c_int, c_int64, c_void_p],
    "qlrt_nf4_linear_group_fwd": [POINTER(NF4Weight), c_int, c_void_p, c_int64, c_void_p, c_void_p, c_int, c_float,
                                  c_void_p, c_void_p, c_void_p, c_void_p],
    "qlrt_nf4_linear_group_bwd": [POINTER(NF4Weight), c_int, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_int, c_float, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_int, c_void_p],
    "qlrt_side_join": [c_void_p],
    "qlrt_side_stream": [c_void_p],
    "qlrt_nf4_gemv": [POINTER(NF4Weight), c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_float, c_void_p, c_void_p, c_void_p],
    "qlrt_gemv_workspace_bytes": [c_int64, c_int64, c_int],
    "qlrt_gemm_bf16": [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int, c_int, c_float, c_int, c_int,
                       c_void_p, c_size_t, c_void_p],
    "qlrt_adam_step": [c_void_p, c_void_p, c_void_p, c_void_p, c_int64] + [c_float] * 8 + [c_void_p, c_void_p],
    "qlrt_adam_step_dev": [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_double, c_void_p,
                           c_void_p],
    "qlrt_sumsq_f64": [c_void_p, c_int64, c_void_p, c_void_p],
    "qlrt_scale_f32": [c_void_p, c_int64, c_float, c_void_p],
    "qlrt_sumsq_f64_pairwise": [c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p,
                                c_void_p],
    "qlrt_prefetch": [c_void_p, c_size_t, c_int, c_void_p],
    "qlrt_rmsnorm_fwd": [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_float, c_void_p],
    "qlrt_rmsnorm_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p],
    "qlrt_add_rmsnorm_fwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_float, c_void_p],
    "qlrt_rmsnorm_bwd_add": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p],
    "qlrt_swiglu_fwd": [c_void_p, c_void_p, c_void_p, c_int64, c_void_p],
    "qlrt_swiglu_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p],
    "qlrt_rope": [c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_int, c_void_p],
    "qlrt_rope_strided": [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int, c_int, c_int, c_int,
                          c_void_p],
    "qlrt_swiglu_cat_fwd": [c_void_p, c_void_p, c_int64, c_int64, c_void_p],
    "qlrt_xent_fwd": [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p],
    "qlrt_xent_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p],
    "qlrt_rope_qkv_fwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_void_p],
    "qlrt_rope_qkv_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_void_p],
    "qlrt_swiglu_cat_bwd": [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p],
    "qlrt_build_info": [],
    "qlrt_set_policy": [ctypes.c_char_p, c_int],
    "qlrt_get_policy": [ctypes.c_char_p, POINTER(c_int)],
}
_RESTYPE = {"qlrt_side_stream": c_void_p, "qlrt_dq_workspace_bytes": c_size_t, "qlrt_linear_workspace_bytes": c_size_t,
            "qlrt_gemv_workspace_bytes": c_size_t,
            "qlrt_nf4_constants_bytes": c_size_t,
            "qlrt_build_info": ctypes.c_char_p}

EXPORTS = tuple(_SIGS)
_lib = None
TORCH_OPS_PATH = os.path.join(os.path.dirname(LIB_PATH), "libqlrt_torch_ops.so")
_ops_loaded = False


def load_torch_ops(path: str = TORCH_OPS_PATH):
    """Register the torch custom ops (``torch.ops.qlrt_b200.*``, CUDA + Meta
    implementations over the same C ABI; csrc/torch_ops.cpp).  Raises if the
    library is missing."""
    global _ops_loaded
    if not _ops_loaded:
        if not os.path.exists(path):
            raise RuntimeError(f"qlrt_b200 torch-op library not built: {path} (run __graft_entry__.build())")
        load_library()
        torch.ops.load_library(path)
        _ops_loaded = True
    return torch.ops.qlrt_b200


def codebook_blob(cb) -> torch.Tensor:
    """A codebook as the qlrt_codebook4 struct bytes (CPU uint8) for the torch ops."""
    return torch.frombuffer(bytearray(bytes(cb.to_c())), dtype=torch.uint8)


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the C ABI.  Raises if the .so is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"qlrt_b200 CUDA library not built: {path} (run __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, c_int)
        _lib = lib
    return _lib


def lib() -> ctypes.CDLL:
    """The library, for a call that will launch kernels: also requires CUDA."""
    if not torch.cuda.is_available():
        raise RuntimeError("qlrt_b200 requires a CUDA (sm_100a) device; there is no CPU fallback")
    return load_library()


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


POLICY_DEFAULT = -0x7FFFFFFF


def set_policy(name: str, value: int | None) -> None:
    """Set an engine launch policy (e.g. "QLRT_STREAMK"); None restores the default."""
    check(load_library().qlrt_set_policy(name.encode(), POLICY_DEFAULT if value is None else int(value)),
          f"set_policy({name})")


def get_policy(name: str) -> int:
    v = c_int()
    check(load_library().qlrt_get_policy(name.encode(), ctypes.byref(v)), f"get_policy({name})")
    return v.value


def check(status: int, what: str) -> None:
    if status == QLRT_OK:
        return
    names = {QLRT_ERR_ARG: "invalid argument", QLRT_ERR_CUDA: "CUDA error",
             QLRT_ERR_UNSUPPORTED: "unsupported shape/layout"}
    if status == QLRT_ERR_ARG:
        raise ValueError(f"{what}: {names[status]}")
    raise RuntimeError(f"{what}: {names.get(status, status)}")
