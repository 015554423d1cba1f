"""Kernel-by-kernel device times of one Cholesky-QR2 call (CUPTI via torch.profiler).

    python tools/diag/qr_kernels.py [m] [n]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1206_3768_b200 as pkg  # noqa: F401
from paper_1206_3768_b200 import linalg

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
n = int(sys.argv[2]) if len(sys.argv) > 2 else 160
torch.cuda.set_device(0)
rng = np.random.default_rng(0)
y0 = torch.from_numpy((rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m)))
                      * np.logspace(0, -1.5, n)[:, None]).cuda().t()
for _ in range(5):
    linalg.qr_orthonormalize_inplace(y0.clone(memory_format=torch.preserve_format))
torch.cuda.synchronize()
y = y0.clone(memory_format=torch.preserve_format)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    linalg.qr_orthonormalize_inplace(y)
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{e.time_range.start - t0:8.1f} us  +{e.time_range.end - e.time_range.start:7.1f} us  {e.name[:90]}")
print(f"span {ev[-1].time_range.end - t0:.1f} us")
