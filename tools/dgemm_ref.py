"""cuBLAS DGEMM throughput on this B200 (context for the fp64 roofline; dev tool)."""
import json
import torch

torch.backends.cuda.matmul.allow_tf32 = False
res = []
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res.append({"probe": "cublas_dgemm", "n": n, "tflops": 2 * n ** 3 / ms / 1e9, "ms": ms})
for r in res:
    print(json.dumps(r))
