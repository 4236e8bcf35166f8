import sys, time, os
sys.path.insert(0, "/root/repo")
import torch, bench, workloads
import paper_0909_4061_b200 as lr
cfg = workloads.CONFIGS[2]
A = bench.build_input(cfg)
host = torch.empty(A.shape, dtype=A.dtype, pin_memory=True); host.copy_(A)
del A; torch.cuda.empty_cache()
for i in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    b, f, _ = lr.randomized_svd(host, cfg.k, cfg.p, cfg.q, cfg.seed, sketch=cfg.sketch, estimate=False)
    dt = time.perf_counter() - t0
    print(f"call {i}: {dt*1e3:.2f} ms", flush=True)
os.environ["LR_OZAKI"] = "0"
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    b, f, _ = lr.randomized_svd(host, cfg.k, cfg.p, cfg.q, cfg.seed, sketch=cfg.sketch, estimate=False)
    print(f"no-ozaki call {i}: {(time.perf_counter()-t0)*1e3:.2f} ms", flush=True)
