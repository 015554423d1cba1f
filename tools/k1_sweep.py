"""K1 throughput sweep vs cuBLAS ZGEMM at the BASELINE filter shapes.

    python tools/k1_sweep.py [--quick]
Prints one JSON line per (n, w): K1 TFLOP/s (fused step, CUDA events over
deg launches) and cuBLAS ZGEMM TFLOP/s for the bare product.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import _lib
from paper_1206_3768_b200._device import Operator, fblock
from paper_1206_3768_b200.chfsi import _filter_into

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true")
ap.add_argument("--bn", type=int, default=0)
a = ap.parse_args()
shapes = [(512, 48), (2048, 160), (2048, 100), (2048, 40), (5000, 600), (5000, 250),
          (12000, 1400)]
if a.quick:
    shapes = shapes[:5]
hcache = {}
for n, w in shapes:
    if n not in hcache:
        hcache.clear()
        g = torch.randn(n, n, dtype=torch.complex128, device="cuda")
        hcache[n] = (g + g.conj().T) / 2
        del g
    h = hcache[n]
    op = Operator(h)
    y = fblock(n, w)
    y.copy_(torch.randn(n, w, dtype=torch.complex128, device="cuda"))
    x = fblock(n, w)
    if a.bn:
        _lib.check(_lib.lib().chfsi_ctx_set_tiling(_lib.ctx(), 64, a.bn, 0))
    win = pkg.FilterWindow(a=-5.0, b=60.0, scale_ref=-70.0)
    deg = 8
    reps = 3 if n <= 5000 else 1
    _filter_into(op, y, x, y, deg, win)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _filter_into(op, y, x, y, deg, win)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (reps * deg)
    yy = torch.randn(n, w, dtype=torch.complex128, device="cuda")
    z = h @ yy
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps * 2):
        z = h @ yy
    e1.record()
    torch.cuda.synchronize()
    ms_c = e0.elapsed_time(e1) / (reps * 2)
    fl = 8.0 * n * n * w
    print(json.dumps({"n": n, "w": w, "k1_us": round(ms * 1e3, 2), "k1_tflops": round(fl / ms / 1e9, 2),
                      "cublas_us": round(ms_c * 1e3, 2), "cublas_tflops": round(fl / ms_c / 1e9, 2)}),
          flush=True)
    _lib.check(_lib.lib().chfsi_ctx_set_tiling(_lib.ctx(), 0, 0, 0))
