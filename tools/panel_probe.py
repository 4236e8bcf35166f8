"""Timing probe of the config-4 panel kernels (m = 2^20, ell = 256): the
m-side apply Y P with a known max|Y| (gemm_f32_pair_kernel, K = 256), the
tcgen05 Gram of the second CholeskyQR pass (lr_gram_tc) and the exact DMMA
Gram (lr_gram).  Run against variant libraries (LOWRANK_B200_LIB=...)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0909_4061_b200 import _lib  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
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
    m, ell = 1 << 20, 256
    g = torch.Generator(device="cuda").manual_seed(0)
    Y = torch.randn(m, ell, device="cuda", generator=g) / 1024
    P = torch.randn(ell, ell, device="cuda", generator=g)
    Q = torch.empty(m, ell, device="cuda")
    G = torch.empty(ell, ell, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    h = _lib.handle()
    out = {"lib": os.path.basename(os.path.dirname(_lib.LIB_PATH))}
    ymax = float(Y.abs().max())
    out["apply_ms"] = timed(lambda: _lib.call(
        "lr_gemm_scaled", h, _lib.F32, _lib.OP_N, m, ell, ell, _lib.ptr(Y), ell, ymax,
        _lib.ptr(P), ell, _lib.ptr(Q), ell))
    out["gram_tc_ms"] = timed(lambda: _lib.call("lr_gram_tc", h, m, ell, _lib.ptr(Y), ell,
                                                _lib.ptr(G), 12, _lib.ptr(st)))
    out["gram_exact_ms"] = timed(lambda: _lib.call("lr_gram", h, _lib.F32, m, ell, _lib.ptr(Y),
                                                   ell, _lib.ptr(G)), reps=3)
    out["hbm_bound_apply_ms"] = 2 * m * ell * 4 / 6.5e12 * 1e3
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in out.items()}),
          flush=True)


if __name__ == "__main__":
    main()
