"""fp64 pass timing: DMMA (lr_gemm) vs the int8-tensor-core emulation
(lr_gemm_ozaki) at the BASELINE configs' fp64 shapes.

    python tools/ozaki_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_0909_4061_b200 import core  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for m, n, ell in [(16384, 8192, 110), (2048, 2048, 30), (16384, 8192, 10), (65536, 4096, 128)]:
    A = torch.randn(m, n, dtype=torch.float64, device="cuda")
    X = torch.randn(n, ell, dtype=torch.float64, device="cuda")
    Z = torch.randn(m, ell, dtype=torch.float64, device="cuda")
    Y = torch.empty(m, ell, dtype=torch.float64, device="cuda")
    W = torch.empty(n, ell, dtype=torch.float64, device="cuda")
    t_prep = timed(lambda: core.ozaki_prepare(A), reps=3)
    oz = core.ozaki_prepare(A)
    flops = 2.0 * m * n * ell
    for adj, (inp, out) in ((False, (X, Y)), (True, (Z, W))):
        t_d = timed(lambda: core.gemm(A, inp, out, adjoint=adj))
        ref = out.clone()
        t_o = timed(lambda: core.ozaki_pass(oz, m, n, inp, out, adj))
        rel = ((out - ref).abs().max() / ref.abs().max()).item()
        print(f"{m}x{n} ell={ell} {'T' if adj else 'N'}: DMMA {t_d * 1e3:8.1f} us "
              f"({flops / t_d / 1e9:6.1f} TF)  int8-emulated {t_o * 1e3:8.1f} us "
              f"({flops / t_o / 1e9:6.1f} TF-equiv, A {m * n * 8 / t_o / 1e6:6.0f} GB/s)  "
              f"max|diff|/max {rel:.1e}", flush=True)
    print(f"  prepare (8 digit planes of A): {t_prep * 1e3:.1f} us")
    del A, oz
    torch.cuda.empty_cache()
