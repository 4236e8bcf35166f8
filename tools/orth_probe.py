"""Development probe: the m-side orthonormalization at config 4's panel shape
(m x 256 fp32, kappa ~ 1e6) -- time per call, status word, loss of
orthogonality and span residual, for LR_SKETCH_QR=0 (exact DMMA Gram) and 1
(sketch-preconditioned, sketch_rows.cu).  Run each setting in its own process:
    LR_SKETCH_QR=0 python tools/orth_probe.py; LR_SKETCH_QR=1 python tools/orth_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0909_4061_b200 import core


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def panel(m, ell, kappa, seed, coherent=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    U = torch.randn(m, ell, device="cuda", dtype=torch.float64, generator=g)
    if coherent:   # a few heavy rows: the hard case for a sparse embedding
        U[:: m // 64] *= 300.0
    U, _ = torch.linalg.qr(U)
    W, _ = torch.linalg.qr(torch.randn(ell, ell, device="cuda", dtype=torch.float64, generator=g))
    s = torch.logspace(0, -torch.log10(torch.tensor(kappa)).item(), ell, device="cuda",
                       dtype=torch.float64)
    return ((U * s) @ W.T).float().contiguous()


for m, ell, kappa, coh in [(1 << 20, 256, 1e6, False), (1 << 20, 256, 1e6, True),
                           (1 << 17, 256, 1e6, False), (1 << 18, 128, 1e3, False),
                           (1 << 20, 256, 1.0, False)]:
    Y = panel(m, ell, kappa, 1, coh)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")

    def run():
        with core.speculate(status):
            return core.orth_dev(Y)

    def run_def():
        with core.speculate(status):
            return core.orth_dev_deferred(Y)

    Q = run()
    torch.cuda.synchronize()
    st = int(status.item())
    Qd = Q.double()
    G = Qd.T @ Qd
    orth = (G - torch.eye(ell, device="cuda", dtype=torch.float64)).abs().max().item()
    Yd = Y.double()
    res = torch.linalg.norm(Yd - Qd @ (Qd.T @ Yd)) / torch.linalg.norm(Yd)
    # upper-triangular R = Q^T Y (the Gram-Schmidt basis): relative size of the strict lower part
    R = Qd.T @ Yd
    low = torch.linalg.norm(torch.tril(R, -1)) / torch.linalg.norm(R)
    t_full = timeit(run)
    t_def = timeit(run_def)
    print(f"m={m} ell={ell} kappa={kappa:g} coherent={coh} sketch={os.environ.get('LR_SKETCH_QR', '1')}: "
          f"status={st} |Q^TQ-I|max={orth:.2e} span res={res.item():.2e} tril(R)={low.item():.2e} "
          f"orth {t_full:.3f} ms deferred {t_def:.3f} ms", flush=True)
    del Y, Q, Qd, Yd
