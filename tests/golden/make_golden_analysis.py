"""Golden rows of the reference's quant_error_report (acceptance criterion 5
input: normal(size=2**17), seed 7).  Run in the build container, where the
reference imports:  python tests/golden/make_golden_analysis.py"""
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from qlrt.analysis import QuantConfig, quant_error_report  # noqa: E402

x = np.random.default_rng(7).normal(size=1 << 17)
cfgs = [QuantConfig("nf4", 64), QuantConfig("fp4-e2m1", 64), QuantConfig("int4", 64),
        QuantConfig("nf4", 64, double_quant=True), QuantConfig("nf-eq4", 64), QuantConfig("nf4", 128)]
rows = quant_error_report(x, cfgs)
out = {"input": "np.random.default_rng(7).normal(size=1 << 17)", "numpy": np.__version__,
       "configs": [[c.codebook, c.blocksize, c.double_quant, c.blocksize2] for c in cfgs],
       "rows": [{"label": r.label, "bits_per_param": r.bits_per_param, "mse": r.mse, "max_abs_err": r.max_abs_err,
                 "entropy_bits": r.entropy_bits, "occupancy": list(r.occupancy)} for r in rows]}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "analysis_report.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(out["rows"], indent=1)[:2000])
