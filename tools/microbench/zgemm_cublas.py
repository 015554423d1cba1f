"""cuBLAS ZGEMM (torch complex128 matmul) at the filter shapes: the library baseline."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
dev = "cuda"
for n, w in [(512, 48), (2048, 160), (5000, 600), (12000, 1400), (8192, 8192)]:
    h = torch.randn(n, n, dtype=torch.complex128, device=dev)
    y = torch.randn(n, w, dtype=torch.complex128, device=dev)
    for _ in range(3):
        z = h @ y
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20 if n <= 5000 else 5
    e0.record()
    for _ in range(reps):
        z = h @ y
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"bench": "cublas_zgemm", "n": n, "w": w, "ms": ms, "tflops": 8.0 * n * n * w / ms / 1e9}))
