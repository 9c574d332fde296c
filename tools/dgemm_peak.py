"""cuBLAS DGEMM (torch.mm f64) throughput on this box: the realism check for the
FP64 roofline denominator.  Not part of the product path."""
import time, torch
dev = torch.device("cuda:0")
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        torch.mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.mm(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"DGEMM n={n}: {2*n**3/best/1e9:.2f} TFLOP/s ({best:.2f} ms)")
    # syrk-ish: a @ a.T
    best = 1e9
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.mm(a, a.T); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"  A@A.T n={n}: {2*n**3/best/1e9:.2f} TFLOP/s full-GEMM-equivalent ({best:.2f} ms)")
