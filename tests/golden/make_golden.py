"""Generate the golden fixtures from the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``qlrt`` from /root/reference/pkg/src (read-only, never copied),
runs the hot-path functions on small seeded inputs and writes
``tests/golden/golden.npz`` + ``tests/golden/golden_meta.json``.  These files
travel to the GPU box; /root/reference does not.  ``tests/test_oracle.py``
pins the CPU oracle against them and the GPU parity tests use them directly.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import qlrt  # noqa: E402
from qlrt import blockquant, codebooks, doublequant, qlora, training  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def h16(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"numpy": np.__version__, "bufsize": int(np.getbufsize()),
                  "qlrt": qlrt.__version__}

    # ---- codebooks -------------------------------------------------------
    for name in ("nf4", "fp4-e2m1", "fp4-e3m0", "int4", "nf-eq4"):
        cb = codebooks.get_codebook(name)
        arrays[f"cb/{name}/values"] = cb.values
        arrays[f"cb/{name}/mids"] = cb.midpoints()
        meta[f"cb/{name}"] = {"n_emitted": cb.n_emitted, "zero_code": cb.zero_code,
                              "values_hex": [float(v).hex() for v in cb.values]}

    # ---- fp8 grid --------------------------------------------------------
    arrays["fp8/decode"] = doublequant.decode_fp8(np.arange(256, dtype=np.uint8))
    rng = np.random.default_rng(11)
    vals, _ = doublequant.Fp8Spec().grid()
    mids = (vals[:-1] + vals[1:]) / 2
    probe = np.concatenate([vals, mids, -mids, rng.normal(scale=100, size=4000),
                            rng.uniform(-1e-3, 1e-3, size=1000),
                            [0.0, -0.0, 480.0, 481.0, 1e6, -1e6, 464.0, -464.0,
                             2.0 ** -10, -(2.0 ** -10), 2.0 ** -11]])
    arrays["fp8/probe"] = probe
    arrays["fp8/probe_codes"] = doublequant.encode_fp8(probe)

    # ---- quantize cases ----------------------------------------------------
    cases = []
    r = np.random.default_rng(0)

    def add_case(tag, x, cb="nf4", bs=64, dq=False, bs2=256):
        q = blockquant.quantize(x, codebooks.get_codebook(cb), blocksize=bs,
                                double_quant=dq, blocksize2=bs2)
        deq = blockquant.dequantize(q)
        arrays[f"q/{tag}/x"] = np.asarray(x)
        arrays[f"q/{tag}/codes"] = q.codes
        if q.constants is not None:
            arrays[f"q/{tag}/constants"] = q.constants
        if q.dq is not None:
            arrays[f"q/{tag}/dq_codes"] = q.dq.codes
            arrays[f"q/{tag}/dq_c1"] = q.dq.c1
            arrays[f"q/{tag}/dq_mu"] = np.array([q.dq.mu], dtype=np.float32)
            arrays[f"q/{tag}/absmax_dq"] = q.block_constants()
        arrays[f"q/{tag}/deq"] = deq
        cases.append({"tag": tag, "codebook": cb, "blocksize": bs, "double_quant": dq,
                      "blocksize2": bs2, "shape": list(np.shape(x))})

    add_case("gauss_f32_dq", r.standard_normal((64, 1024), dtype=np.float32), dq=True)
    add_case("gauss_f32_plain", r.standard_normal((32, 512), dtype=np.float32))
    add_case("llama_like", (0.02 * r.standard_normal((128, 11008 // 8))).astype(np.float32), dq=True)
    odd = r.standard_normal(64 * 37 + 13).astype(np.float32)
    add_case("ragged_dq", odd, dq=True)
    z = r.standard_normal(64 * 300).astype(np.float32)
    z[64 * 5:64 * 9] = 0.0           # whole zero blocks
    z[r.choice(z.size, 500, replace=False)] = 0.0
    add_case("zero_blocks_dq", z, dq=True)
    # exact midpoints / ties: values = mid * c for a block whose absmax is 1
    cb = codebooks.get_codebook("nf4")
    m = cb.midpoints()
    tie = np.concatenate([[1.0], m, -m, [-1.0], np.zeros(64 - 2 - 2 * m.size)]).astype(np.float64)
    add_case("ties_f64", tie)
    add_case("bs16", r.standard_normal(16 * 50), bs=16)
    add_case("bs2_100", r.standard_normal(64 * 700).astype(np.float32), dq=True, bs2=100)
    add_case("int4_table", r.standard_normal(64 * 40).astype(np.float32), cb="int4")
    add_case("fp4_table", r.standard_normal(64 * 40).astype(np.float32), cb="fp4-e2m1")
    add_case("nfeq4_zero", np.concatenate([np.zeros(64), r.standard_normal(128)]), cb="nf-eq4")
    add_case("single", np.array([0.7]), dq=False)
    add_case("bf16_grid", _bf16_values(r.standard_normal(64 * 64).astype(np.float32)), dq=True)
    meta["quant_cases"] = cases

    # ---- DQ mean order: adversarial constants ---------------------------
    dq_cases = []
    for i, n in enumerate([5, 100, 129, 1000, 8192, 8193, 20000, 70001]):
        rr = np.random.default_rng(100 + i)
        c = np.abs(rr.standard_normal(n) * np.exp(rr.uniform(-30, 30, size=n))).astype(np.float32)
        dq = doublequant.dq_compress(c, blocksize2=256)
        arrays[f"dq/{i}/c"] = c
        arrays[f"dq/{i}/mu"] = np.array([dq.mu], dtype=np.float32)
        arrays[f"dq/{i}/c1"] = dq.c1
        arrays[f"dq/{i}/codes"] = dq.codes
        arrays[f"dq/{i}/rec"] = doublequant.dq_decompress(dq)
        arrays[f"dq/{i}/sum64"] = np.array([c.sum(dtype=np.float64)])
        dq_cases.append(n)
    meta["dq_cases"] = dq_cases

    # ---- QLinear (float64 mode over a bf16-representable dense base) ------
    ql = []
    for i, (mm, kk, nn, rank) in enumerate([(4, 64, 128, 8), (33, 128, 192, 16), (256, 256, 512, 64)]):
        rr = np.random.default_rng(200 + i)
        w = (0.02 * rr.standard_normal((kk, nn))).astype(np.float32)
        q = blockquant.quantize(w, codebooks.get_codebook("nf4"), 64, double_quant=True)
        wdq = _bf16_values(blockquant.dequantize(q).astype(np.float32)).astype(np.float64)
        ad = qlora.lora_init(kk, nn, rank, 16.0, rr, dtype=np.float64)
        ad.l1 = _bf16_values(ad.l1.astype(np.float32)).astype(np.float64)
        ad.l2 = _bf16_values((0.01 * rr.standard_normal((rank, nn))).astype(np.float32)).astype(np.float64)
        x = _bf16_values(rr.standard_normal((mm, kk)).astype(np.float32)).astype(np.float64)
        dy = _bf16_values(rr.standard_normal((mm, nn)).astype(np.float32)).astype(np.float64)
        lin = qlora.QLinear(wdq, adapters=[ad], dtype=np.float64)
        y, cache = lin.forward(x)
        dx, grads = lin.backward(dy, cache)
        for key, val in (("w", w), ("x", x), ("dy", dy), ("l1", ad.l1), ("l2", ad.l2),
                         ("y", y), ("dx", dx), ("dl1", grads["adapter0.l1"]),
                         ("dl2", grads["adapter0.l2"]), ("codes", q.codes),
                         ("dq_codes", q.dq.codes), ("dq_c1", q.dq.c1),
                         ("dq_mu", np.array([q.dq.mu], dtype=np.float32))):
            arrays[f"ql/{i}/{key}"] = val
        ql.append({"m": mm, "k": kk, "n": nn, "rank": rank, "alpha": 16.0})
    meta["qlinear_cases"] = ql

    # ---- Adam (fp32, NEP 50 constant rounding) ----------------------------
    rr = np.random.default_rng(300)
    p = rr.standard_normal(1000).astype(np.float32)
    cfg = training.TrainConfig(learning_rate=0.01)
    opt = training.AdamOptimizer({"p": p}, cfg, training.PlainMomentStore())
    arrays["adam/p0"] = p.copy()
    for t in range(5):
        g = (rr.standard_normal(1000) * 10 ** rr.uniform(-6, 1, size=1000)).astype(np.float32)
        arrays[f"adam/g{t}"] = g
        opt.step({"p": g})
        arrays[f"adam/p{t + 1}"] = p.copy()
    grads = {"a": (rr.standard_normal(300)).astype(np.float32),
             "b": (rr.standard_normal(77)).astype(np.float32)}
    arrays["clip/a"], arrays["clip/b"] = grads["a"].copy(), grads["b"].copy()
    norm = training.clip_global_norm(grads, ["a", "b"], 0.3)
    arrays["clip/a_out"], arrays["clip/b_out"] = grads["a"], grads["b"]
    meta["clip_norm"] = norm

    # ---- config C1 hashes ------------------------------
    x = np.random.default_rng(0).standard_normal((4096, 4096), dtype=np.float32)
    q = blockquant.quantize(x.astype(np.float64), codebooks.get_codebook("nf4"), 64,
                            double_quant=True, blocksize2=256)
    deq32 = blockquant.dequantize(q).astype(np.float32)
    plain = blockquant.quantize(x.astype(np.float64), codebooks.get_codebook("nf4"), 64)
    meta["c1"] = {"x": h16(x), "codes": h16(q.codes), "dq_codes": h16(q.dq.codes),
                  "dq_c1": h16(q.dq.c1), "mu_hex": float(q.dq.mu).hex(),
                  "plain_constants": h16(plain.constants), "deq_f32": h16(deq32),
                  "absmax_dq": h16(q.block_constants())}
    try:
        import torch
        meta["c1"]["deq_bf16"] = h16(torch.from_numpy(deq32).to(torch.bfloat16)
                                     .view(torch.int16).numpy())
    except Exception:  # pragma: no cover
        pass

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays;", json.dumps(meta["c1"]))


def _bf16_values(a: np.ndarray) -> np.ndarray:
    """float32 -> nearest bf16 (RNE) -> float32, without torch."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


if __name__ == "__main__":
    main()
