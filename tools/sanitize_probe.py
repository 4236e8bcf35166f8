"""Small invocations of every TMA / tcgen05 / mbarrier kernel family, for
compute-sanitizer (racecheck, synccheck) runs:

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py

Shapes are tiny so the instrumented run finishes in minutes; each kernel is
checked against an fp64 product as well (a race that corrupts data fails)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0909_4061_b200 import _lib, core, sketch  # noqa: E402
from paper_0909_4061_b200 import factor  # noqa: E402


def check(name, got, ref, tol):
    err = float((got.double() - ref).abs().max() / max(ref.abs().max().item(), 1e-300))
    print(f"{name}: rel err {err:.2e}", flush=True)
    assert err <= tol, name


g = torch.Generator(device="cuda").manual_seed(0)


def f32pass(m, n, ell, env):
    for k, v in env.items():
        os.environ[k] = v
    A = torch.randn(m, n, device="cuda", generator=g)
    X = torch.randn(n, ell, device="cuda", generator=g)
    Y = torch.empty(m, ell, device="cuda")
    core._pass(A, X, Y, False, float(A.abs().max()))
    check(f"f32 AX {m}x{n}x{ell} {env}", Y, A.double() @ X.double(), 1e-5)
    W = torch.randn(m, ell, device="cuda", generator=g)
    Z = torch.empty(n, ell, device="cuda")
    core._pass(A, W, Z, True, float(A.abs().max()))
    check(f"f32 ATY {m}x{n}x{ell} {env}", Z, A.double().T @ W.double(), 1e-5)
    for k in env:
        del os.environ[k]


f32pass(512, 384, 64, {"LR_TC_PAIR": "0", "LR_TC_M256": "0"})     # single-CTA kernel
f32pass(2048, 512, 96, {})                                          # m256 (deep K) / pair
f32pass(1024, 256, 64, {"LR_TC_PAIR": "1"})                        # CTA-pair kernel
Y = torch.randn(4096, 200, device="cuda", generator=g) / 64
G = torch.empty(200, 200, dtype=torch.float64, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
_lib.call("lr_gram_tc", _lib.handle(), 4096, 200, _lib.ptr(Y), 200, _lib.ptr(G), 12, _lib.ptr(st))
check("gram_tc 4096x200", G, Y.double().T @ Y.double(), 1e-5)
for rows in (1024, 8192):                                           # int8 fp64: single / pair
    A = torch.randn(rows, 512, dtype=torch.float64, device="cuda", generator=g)
    X = torch.randn(512, 60, dtype=torch.float64, device="cuda", generator=g)
    oz = core.ozaki_prepare(A)
    Yo = torch.empty(rows, 60, dtype=torch.float64, device="cuda")
    core.ozaki_pass(oz, rows, 512, X, Yo, False)
    check(f"ozaki {rows}", Yo, A @ X, 1e-13)
A = torch.randn(4096, 1024, dtype=torch.float64, device="cuda", generator=g)
X = torch.randn(1024, 64, dtype=torch.float64, device="cuda", generator=g)
Yd = torch.empty(4096, 64, dtype=torch.float64, device="cuda")
core.gemm(A, X, Yd)
check("dmma tma", Yd, A @ X, 1e-13)
Ac = torch.randn(64, 1024, dtype=torch.complex64, device="cuda", generator=g)
op = sketch.srft_operator(1024, 24, 1)
Ys = sketch.srft_dev(Ac, op)
print("srft16 ok", Ys.shape, flush=True)
M = np.random.default_rng(1).standard_normal((300, 8))
f = factor.row_id(M, 8)
print("row_id ok", np.abs(f.X).max() <= 2 + 1e-10, flush=True)
torch.cuda.synchronize()
print("sanitize probe done", flush=True)
