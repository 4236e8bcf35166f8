"""Config-4 numerics on the GPU at one 65536-row block, against the
reference's fp64 run (tests/golden/cfg4s.npz): the first index j whose
sigma_j misses 1e-4 relative, and the relative errors of the leading sigma,
for the arithmetic variants selected by environment variables
(LR_F32_SIMT=1: honest fp32 FFMA passes; LR_TC_M256 / LR_TC_PAIR /
LR_GRAM_TC: kernel choices).  Prints one JSON line."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0909_4061_b200 as lr  # noqa: E402
import workloads  # noqa: E402
from paper_0909_4061_b200 import _lib  # noqa: E402

g = dict(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "cfg4s.npz")))
c = workloads.CONFIGS[4]
A, _ = workloads.build_cfg4_host(m=65536)
if os.environ.get("LR_F32_SIMT") == "1":
    _lib.set_f32_mode(_lib.F32_SIMT)
basis, f, est = lr.randomized_svd(A, c.k, c.p, c.q, c.seed)
s_ref = g["sigma"]
rel = np.abs(np.asarray(f.sigma) - s_ref) / s_ref
bad = np.nonzero(rel > 1e-4)[0]
print(json.dumps({"variant": os.environ.get("VARIANT", "default"),
                  "first_violation_j": int(bad[0]) + 1 if bad.size else None,
                  "sigma_ref_at_violation": float(s_ref[bad[0]] / s_ref[0]) if bad.size else None,
                  "rel_top5": [float(x) for x in rel[:5]],
                  "rel_max_j_le_100": float(rel[:100].max()),
                  "rel_max_j_le_120": float(rel[:120].max()),
                  "est_rel": float(abs(est - g["est"][0]) / g["est"][0])}), flush=True)
