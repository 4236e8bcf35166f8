"""Diagnostics: one cfg2 rSVD step with the speculative flags printed and
per-call wall/GPU timings (development tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_0909_4061_b200 as lr
from paper_0909_4061_b200 import core
cfg = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
A, _ = workloads.build_synthetic_device(cfg.m, cfg.n, workloads.spectrum(cfg.idx, cfg.n), cfg.seed)
op = lr.DenseOperator(A)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for it in range(3):
    st.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with core.speculate(st):
        Q = lr.rangefinder.subspace_iteration_range_dev(op, cfg.ell, cfg.q, cfg.seed)
        t1 = time.perf_counter()
        U, S, V = lr.factor.direct_svd_dev(op, Q)
        t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"iter {it}: status={int(st.item())} enqueue stageA {1e3*(t1-t0):.2f} ms, stageB {1e3*(t2-t1):.2f} ms, total wall {1e3*(t3-t0):.2f} ms", flush=True)
# per-kernel-class GPU timing with events
def timed(fn, *a):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record(); r = fn(*a); e.record(); torch.cuda.synchronize()
    return r, s.elapsed_time(e)
Y = torch.randn(cfg.m, cfg.ell, dtype=torch.float64, device="cuda")
with core.speculate(st):
    for _ in range(2):
        _, t = timed(core.orth_dev, Y)
    print(f"orth_fast {cfg.m}x{cfg.ell}: {t:.3f} ms")
    Z = torch.randn(cfg.n, cfg.ell, dtype=torch.float64, device="cuda")
    for _ in range(2):
        _, t = timed(core.small_svd_from_adjoint, Z.clone())
    print(f"small_svd_fast {cfg.n}x{cfg.ell}: {t:.3f} ms  status={int(st.item())}")
G = torch.empty(cfg.ell, cfg.ell, dtype=torch.float64, device="cuda")
h = lr._lib.handle()
for _ in range(2):
    _, t = timed(lambda: lr._lib.call("lr_gram", h, 1, cfg.m, cfg.ell, lr._lib.ptr(Y), cfg.ell, lr._lib.ptr(G)))
print(f"gram: {t:.3f} ms")
P = torch.empty_like(G); R = torch.empty_like(G); info = torch.zeros(4, dtype=torch.int32, device="cuda")
G2 = (Y.T @ Y).contiguous()
for _ in range(2):
    _, t = timed(lambda: lr._lib.call("lr_chol_drop", h, 1, cfg.ell, lr._lib.ptr(G2), 1e-10, 1e-13, 0.0, lr._lib.ptr(P), lr._lib.ptr(R), lr._lib.ptr(info)))
print(f"chol: {t:.3f} ms")
Rm = torch.triu(torch.randn(cfg.ell, cfg.ell, dtype=torch.float64, device="cuda")) + 10 * torch.eye(cfg.ell, dtype=torch.float64, device="cuda")
Wj = torch.empty_like(Rm); Jj = torch.empty_like(Rm); Sj = torch.empty(cfg.ell, dtype=torch.float64, device="cuda")
for _ in range(2):
    _, t = timed(lambda: lr._lib.call("lr_jacobi_svd", h, 1, cfg.ell, lr._lib.ptr(Rm), lr._lib.ptr(Wj), lr._lib.ptr(Sj), lr._lib.ptr(Jj), lr._lib.ptr(info)))
print(f"jacobi: {t:.3f} ms sweeps={int(info[0].item())}")
X = torch.randn(cfg.n, cfg.ell, dtype=torch.float64, device="cuda")
Yo = torch.empty(cfg.m, cfg.ell, dtype=torch.float64, device="cuda")
for _ in range(3):
    _, t = timed(lambda: core.gemm(A, X, Yo))
print(f"pass N: {t:.3f} ms")
for _ in range(3):
    _, t = timed(lambda: core.gemm(A, Yo, X, adjoint=True))
print(f"pass T: {t:.3f} ms")
if lr._lib.HOST_PROFILE is not None:
    lr._lib.HOST_PROFILE.clear()
    st.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with core.speculate(st):
        Q = lr.rangefinder.subspace_iteration_range_dev(op, cfg.ell, cfg.q, cfg.seed)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"stage A enqueue {1e3*(t1-t0):.2f} ms; per-call host time:")
    for k, (c, s) in sorted(lr._lib.HOST_PROFILE.items(), key=lambda x: -x[1][1]):
        print(f"  {k:24s} {c:4d} calls {1e3*s:8.3f} ms  ({1e6*s/c:.1f} us/call)")
