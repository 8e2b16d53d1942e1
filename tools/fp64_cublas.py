"""cuBLAS DGEMM / ZGEMM throughput on the box (the FP64 roofline denominator
for the front factorisation; MEASURED_PEAKS.json has no FP64 figure)."""
import torch

for dt, name, fpm in ((torch.float64, "DGEMM", 2), (torch.complex128, "ZGEMM", 8)):
    for n in (2048, 4096, 8192):
        a = torch.randn(n, n, dtype=dt, device="cuda")
        b = torch.randn(n, n, dtype=dt, device="cuda")
        for _ in range(2):
            a @ b
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(5):
            e0.record()
            a @ b
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{name} n={n}: {fpm * n**3 / best / 1e9:.2f} TFLOP/s (real flops)", flush=True)
