"""Timing probe of the fp32 tensor-core pass kernel at the config-4 shape
(2^20 x 4096, ell = 256): A X and A^T Y passes, the m x 256 . 256 x 256
apply, and the fp64-accumulated Gram of an m x 256 panel.  Run against a
variant library with LOWRANK_B200_LIB=... (tools/tc_variants.sh builds the
LR_TC_DBG timing variants)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0909_4061_b200 import _lib, core  # noqa: E402


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    m, n, ell = 1 << 20, 4096, 256
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(m, n, device="cuda", generator=g)
    X = torch.randn(n, ell, device="cuda", generator=g)
    Yt = torch.randn(m, ell, device="cuda", generator=g) / 1024
    P = torch.randn(ell, ell, device="cuda", generator=g)
    Y = torch.empty(m, ell, device="cuda")
    Z = torch.empty(n, ell, device="cuda")
    amax = float(A.abs().max())
    out = {"lib": os.path.basename(os.path.dirname(_lib.LIB_PATH))}
    out["AX_ms"] = timed(lambda: core._pass(A, X, Y, False, amax))
    out["ATY_ms"] = timed(lambda: core._pass(A, Yt, Z, True, amax))
    out["apply_ms"] = timed(lambda: core.gemm_dev(Yt, P, Y))
    G = torch.empty(ell, ell, dtype=torch.float64, device="cuda")
    h = _lib.handle()
    out["gram_ms"] = timed(lambda: _lib.call("lr_gram", h, _lib.F32, m, ell, _lib.ptr(Yt),
                                             ell, _lib.ptr(G)))
    fl = 3 * 2.0 * m * n * ell
    out["AX_tflops_issued"] = fl / out["AX_ms"] / 1e9
    out["ATY_tflops_issued"] = fl / out["ATY_ms"] / 1e9
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in out.items()}),
          flush=True)


if __name__ == "__main__":
    main()
