"""Run the K1 fused Chebyshev step at a BASELINE shape (for ncu captures).

    python tools/profile_k1.py --n 2048 --w 160 --deg 16 --reps 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200._device import Operator, fblock
from paper_1206_3768_b200.chfsi import _filter_into
from paper_1206_3768_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--w", type=int, default=160)
ap.add_argument("--deg", type=int, default=16)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--variant", default="auto")
ap.add_argument("--split", type=int, default=0, help="grid override (148: one chain of the two-chain filter)")
a = ap.parse_args()
torch.manual_seed(0)
g = torch.randn(a.n, a.n, dtype=torch.complex128, device="cuda")
h = (g + g.conj().T) / 2
del g
op = Operator(h)
if a.variant != "auto" or a.split:
    bm, bn = (64, 32) if a.variant == "auto" else (int(t) for t in a.variant.split("x"))
    _lib.check(_lib.lib().chfsi_ctx_set_tiling(_lib.ctx(), bm, bn, a.split))
y = fblock(a.n, a.w)
y.copy_(torch.randn(a.n, a.w, dtype=torch.complex128, device="cuda"))
x = fblock(a.n, a.w)
win = pkg.FilterWindow(a=-5.0, b=60.0, scale_ref=-70.0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
_filter_into(op, y, x, y, a.deg, win)
torch.cuda.synchronize()
e0.record()
for _ in range(a.reps):
    _filter_into(op, y, x, y, a.deg, win)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / (a.reps * a.deg)
fl = 8.0 * a.n * a.n * a.w
print(f"n={a.n} w={a.w}: {ms*1e3:.1f} us per step, {fl / ms / 1e9:.2f} TFLOP/s")
