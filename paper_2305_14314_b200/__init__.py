"""paper_2305_14314_b200: B200-native (sm_100a) QLoRA hot path behind the API of
the reference package ``qlrt`` 0.1.0.

Drop-in surface (reference names, GPU tensors):
  codebooks   get_codebook, make_nf_codebook, Codebook, inv_normal_cdf
  blockquant  quantize, dequantize, pack_codes, unpack_codes, BlockQuantized
  doublequant dq_compress, dq_decompress, encode_fp8, decode_fp8, DQConstants,
              Fp8Spec, bits_per_param
  qlora       QLinear, LoraAdapter, lora_init
  training    AdamOptimizer, TrainConfig, clip_global_norm, PlainMomentStore,
              PagedMomentStore
  paging      Pager, PagerConfig, pager_open
  parallel    GradBucket, allreduce_mean (data-parallel adapter gradients)
  analysis    quant_error_report, QuantConfig, QuantErrorRow (data-type comparison)
  container   save, load, inspect_header (.qlrt v1, byte-compatible, GPU tensors)
  llama       LlamaConfig, LlamaQLoRA (LLaMA-shaped QLoRA harness, C3/C5)

Every computation runs in the CUDA library ``_lib/libqlrt_b200.so``
(hand-written sm_100a kernels, C ABI in include/qlrt_b200.h).  There is no CPU
fallback: calls raise RuntimeError without the library or a GPU.
"""

from ._native import EXPORTS, LIB_PATH, get_policy, load_library, set_policy
from . import container
from .analysis import QuantConfig, QuantErrorRow, quant_error_report
from .blockquant import BlockQuantized, dequantize, pack_codes, quantize, unpack_codes
from .codebooks import (CODEBOOK_NAMES, Codebook, get_codebook, inv_normal_cdf, make_fp4_codebook,
                        make_int_codebook, make_nf_codebook, make_nf_midpoint_codebook)
from .doublequant import DQConstants, Fp8Spec, bits_per_param, decode_fp8, dq_compress, dq_decompress, encode_fp8
from .errors import (BadMagicError, ChecksumMismatchError, ContainerError, CorruptDataError, QlrtError,
                     TrainingDivergedError, TruncatedFileError, UnsupportedVersionError)
from .paging import Pager, PagerConfig, Slab, pager_open
from .parallel import GradBucket, allreduce_mean
from .qlora import PLACEMENTS, LoraAdapter, QLinear, QLinearGroup, gemm_bf16, lora_init, side_join
from .training import AdamOptimizer, PagedMomentStore, PlainMomentStore, TrainConfig, clip_global_norm
from . import toy

__version__ = "0.1.0"
