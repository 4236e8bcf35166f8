"""cuBLASLt int8 / bf16 GEMM throughput on this GPU (reference points for the
int8-emulated fp64 passes)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import torch  # noqa: E402

print(f"int8 (torch._int_mm 8192^3): {bench.measured_int8_peak():.0f} TOP/s")
for n, k in ((16384, 8192), (8192, 8192)):
    a = torch.randint(-64, 64, (n, k), dtype=torch.int8, device="cuda")
    b = torch.randint(-64, 64, (k, 128), dtype=torch.int8, device="cuda")
    for _ in range(3):
        torch._int_mm(a, b)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        torch._int_mm(a, b)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 10 / 1e3
    print(f"int8 {n}x{k}x128: {2.0 * n * k * 128 / t / 1e12:.0f} TOP/s")
