"""Measure cuBLAS DGEMM (torch.matmul float64) burst throughput: the FP64 roofline denominator."""
import json, sys, torch
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[n] = 2 * n ** 3 / (best * 1e-3) / 1e12
    print(f"DGEMM n={n}: {res[n]:.2f} TFLOP/s ({best:.2f} ms)")
print(json.dumps({"dgemm_tflops": res}))
