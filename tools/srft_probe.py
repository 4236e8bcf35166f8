"""Timing of the SRFT sketch at the config-3 shape (8192 x 8192 complex64,
ell = 120) for the three device paths (LR_SRFT unset: radix-16 Stockham FFT;
=radix2: the round-1 radix-2 kernel; =gemm: the dense picked-DFT-columns pass
on the tensor cores).  Prints one JSON line; HBM bound = A bytes / peak."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0909_4061_b200 import sketch  # noqa: E402


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


out = {}
for dt in (torch.complex64, torch.complex128):
    n = 8192
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(n, n, dtype=dt, device="cuda", generator=g)
    op = sketch.srft_operator(n, 120, 3)
    amax = float(A.abs().max())
    for mode in ("fft16", "radix2", "gemm"):
        os.environ["LR_SRFT"] = "" if mode == "fft16" else mode
        if dt == torch.complex128 and mode == "gemm":
            continue
        ms = timed(lambda: sketch.srft_dev(A, op, amax=amax))
        out[f"{str(dt).split('.')[-1]}_{mode}_ms"] = round(ms, 4)
    out[f"{str(dt).split('.')[-1]}_hbm_bound_ms"] = round(A.numel() * A.element_size() / 6.5485e12 * 1e3, 4)
    del A
print(json.dumps(out), flush=True)
