"""Time back_transform (x = L^-H y) at C2/C3 shapes, CUDA events + wall."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1206_3768_b200 as pkg

for n, nev in ((2048, 128), (5000, 500)):
    c = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    b = torch.eye(n, dtype=torch.complex128, device="cuda") + c @ c.conj().T / (4 * n)
    l = torch.linalg.cholesky(b).t().contiguous().t()
    y = torch.randn(n, nev, dtype=torch.complex128, device="cuda").t().contiguous().t()
    sol = pkg.EigenSolution(values=np.zeros(nev), vectors=y)
    for _ in range(3):
        pkg.back_transform(l, sol)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(10):
        pkg.back_transform(l, sol)
    e1.record()
    torch.cuda.synchronize()
    print(n, nev, "device ms", e0.elapsed_time(e1) / 10, "wall ms", (time.perf_counter() - t0) * 100)
