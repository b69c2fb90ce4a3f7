"""quant_error_report on the GPU kernels vs the reference's own rows
(tests/golden/analysis_report.json, made by make_golden_analysis.py), and
acceptance criterion 5 (pkg/tests/test_acceptance.py:122-136) through the
sm_100a quantize / dequantize path."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_report_matches_reference_rows(qb, cuda):
    from paper_2305_14314_b200.analysis import QuantConfig, quant_error_report
    g = json.load(open(os.path.join(HERE, "golden", "analysis_report.json")))
    x = np.random.default_rng(7).normal(size=1 << 17)
    cfgs = [QuantConfig(c, b, dq, b2) for c, b, dq, b2 in g["configs"]]
    rows = quant_error_report(x, cfgs)
    for r, want in zip(rows, g["rows"]):
        assert r.label == want["label"]
        assert r.bits_per_param == want["bits_per_param"]
        assert list(r.occupancy) == want["occupancy"], r.label          # codes bit-exact
        assert r.max_abs_err == want["max_abs_err"], r.label            # dequant bit-exact
        assert abs(r.mse - want["mse"]) <= 1e-12 * want["mse"], r.label  # summation order differs
        assert abs(r.entropy_bits - want["entropy_bits"]) <= 1e-12 * want["entropy_bits"], r.label


def test_acceptance_criterion_5_dtype_ordering(qb, cuda):
    from paper_2305_14314_b200.analysis import QuantConfig, quant_error_report
    x = np.random.default_rng(7).normal(size=1 << 17)
    nf4, fp4, int4, dq = quant_error_report(x, [QuantConfig("nf4", 64), QuantConfig("fp4-e2m1", 64),
                                               QuantConfig("int4", 64), QuantConfig("nf4", 64, double_quant=True)])
    assert nf4.mse < fp4.mse and nf4.mse < int4.mse and dq.mse / nf4.mse <= 1.05
