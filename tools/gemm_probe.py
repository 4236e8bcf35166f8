"""Development probe: device time of the fp64 pass GEMMs at config-2 shapes
(A 16384 x 8192, ell = 110): A X (NN) and A^T Y (TN), CUDA-graph timed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0909_4061_b200 import _lib, core


def timeit(fn, reps=10):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn(); fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st, capture_error_mode="relaxed"):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); g.replay(); e.record()
        torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


m, n = int(os.environ.get("M", 16384)), int(os.environ.get("N", 8192))
A = torch.randn(m, n, dtype=torch.float64, device="cuda")
for ell in [int(x) for x in os.environ.get("ELLS", "110,30,128").split(",")]:
    X = torch.randn(n, ell, dtype=torch.float64, device="cuda")
    Q = torch.randn(m, ell, dtype=torch.float64, device="cuda")
    Y = torch.empty(m, ell, dtype=torch.float64, device="cuda")
    Z = torch.empty(n, ell, dtype=torch.float64, device="cuda")
    tn = timeit(lambda: core.gemm(A, X, Y))
    tt = timeit(lambda: core.gemm(A, Q, Z, adjoint=True))
    fl = 2.0 * m * n * ell
    ref = A @ X
    err = (Y - ref).abs().max().item() / ref.abs().max().item()
    print(f"ell={ell}: NN {tn:.3f} ms ({fl / tn / 1e9:.1f} TF)  TN {tt:.3f} ms "
          f"({fl / tt / 1e9:.1f} TF)  err {err:.1e}", flush=True)
