"""cuBLAS DGEMM yardstick (torch.matmul float64) on B200 — context only, never on the product path."""
import json
import torch

torch.backends.cuda.matmul.allow_tf32 = False
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"kernel": "cublas_dgemm", "n": n, "ms": best, "tflops": 2 * n**3 / best / 1e9}))
m = n = 1408; k = 1982464 // 8
a = torch.randn(m, k, dtype=torch.float64, device="cuda")
b = torch.randn(k, n, dtype=torch.float64, device="cuda")
c = a @ b; torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(json.dumps({"kernel": "cublas_dgemm_thin", "m": m, "n": n, "k": k, "ms": ms, "tflops": 2 * m * n * k / ms / 1e9}))
