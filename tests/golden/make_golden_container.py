"""Reference-written .qlrt files (pkg/src/qlrt/container.py save) for the
byte-compatibility tests, plus each file's dequantized float64 array.  Run in
the build container, where the reference imports:
    python tests/golden/make_golden_container.py"""
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from qlrt import container  # noqa: E402
from qlrt.blockquant import dequantize, quantize  # noqa: E402
from qlrt.codebooks import get_codebook  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "containers")
CASES = {  # name: (seed, shape, codebook, blocksize, dq)
    "golden_nf4_dq": (42, (8, 16), "nf4", 64, True),     # test_container.py save_golden
    "nf4_plain_64x64": (1, (64, 64), "nf4", 64, False),
    "nf4_dq_ragged": (2, (3, 100), "nf4", 64, True),
    "int4_plain": (3, (1000,), "int4", 64, False),
    "fp4_dq": (4, (32, 96), "fp4-e2m1", 64, True),
    "nfeq4_b16": (5, (7, 9), "nf-eq4", 16, False),
    "scalar": (6, (), "nf4", 64, False),
    # k != 4: one byte per code (container.py:180-181)
    "nf3_plain": (7, (5, 40), "nf3", 64, False),
    "int8_dq": (8, (300,), "int8", 64, True),
    "int2_b32": (9, (3, 33), "int2", 32, False),
}
arrays = {}
for name, (seed, shape, cb, bs, dq) in CASES.items():
    x = np.random.default_rng(seed).normal(size=shape) if shape else np.float64(np.random.default_rng(seed).normal())
    q = quantize(np.asarray(x), get_codebook(cb), blocksize=bs, double_quant=dq)
    container.save(q, os.path.join(OUT, name + ".qlrt"))
    arrays[name + "/x"] = np.asarray(x, dtype=np.float64)
    arrays[name + "/deq"] = dequantize(q)
np.savez_compressed(os.path.join(OUT, "arrays.npz"), **arrays)
print(sorted(os.listdir(OUT)))
