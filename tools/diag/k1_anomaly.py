"""K1 time across (n, w, grid) to map slow schedule regimes.

    python tools/diag/k1_anomaly.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import _lib
from paper_1206_3768_b200._device import Operator, fblock
from paper_1206_3768_b200.chfsi import _filter_into


def timed(fn, reps=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cases = [(n, 160, 32, s) for n in (3072, 3584, 4096, 4608, 5120) for s in (0, 148)]
cases += [(4096, w, 32, 0) for w in (96, 128, 192, 224)]
cases += [(4096, 160, 32, s) for s in (200, 250, 280)]
win = pkg.FilterWindow(a=-5.0, b=60.0, scale_ref=-70.0)
hc = {}
for n, w, bn, split in cases:
    if n not in hc:
        hc.clear()
        g = torch.randn(n, n, dtype=torch.complex128, device="cuda")
        hc[n] = (g + g.conj().T) / 2
    op = Operator(hc[n])
    y = fblock(n, w)
    y.copy_(torch.randn(n, w, dtype=torch.complex128, device="cuda"))
    x = fblock(n, w)
    _lib.check(_lib.lib().chfsi_ctx_set_tiling(_lib.ctx(), 64, bn, split))
    ms = timed(lambda: _filter_into(op, y, x, y, 8, win)) / 8
    print(json.dumps({"n": n, "w": w, "bn": bn, "grid": split, "us": round(ms * 1e3, 1),
                      "tflops": round(8.0 * n * n * w / ms / 1e9, 2)}), flush=True)
_lib.check(_lib.lib().chfsi_ctx_set_tiling(_lib.ctx(), 0, 0, 0))
