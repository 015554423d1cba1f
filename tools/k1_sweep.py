"""K1 throughput sweep vs cuBLAS ZGEMM at the BASELINE filter shapes.

    python tools/k1_sweep.py [--quick] [--variants auto,64x32,32x32,...]
Prints one JSON line per (n, w, variant): K1 TFLOP/s (fused step, CUDA
events over deg launches) and cuBLAS ZGEMM TFLOP/s for the bare product.
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
ap.add_argument("--variants", default="auto")
ap.add_argument("--shapes", default="")
ap.add_argument("--no-cublas", action="store_true")
ap.add_argument("--chains", default="2", help="filter launch chains for the auto tiling (1, 2 or 1,2)")
ap.add_argument("--products", default="3,4", help="K1 complex products to compare (3 = Gauss/3M, 4 = 4M)")
a = ap.parse_args()
shapes = [(512, 48), (2048, 160), (2048, 100), (2048, 40), (5000, 600), (5000, 250),
          (12000, 1400)]
if a.shapes:
    shapes = [tuple(int(v) for v in s.split("x")) for s in a.shapes.split(",")]
if a.quick:
    shapes = shapes[:5]
variants = a.variants.split(",")


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


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
    win = pkg.FilterWindow(a=-5.0, b=60.0, scale_ref=-70.0)
    deg = 8
    reps = 3 if n <= 5000 else 1
    cub = None
    if not a.no_cublas:
        yy = torch.randn(n, w, dtype=torch.complex128, device="cuda")
        ms_c = timed(lambda: h @ yy, reps * 2)
        cub = 8.0 * n * n * w / ms_c / 1e9
    for v, prod, ch in [(v, pr, ch) for v in variants for pr in a.products.split(",")
                        for ch in (a.chains.split(",") if v == "auto" else ["1"])]:
        _lib.lib().chfsi_set_complex_product(int(prod))
        _lib.check(_lib.lib().chfsi_ctx_set_filter_chains(_lib.ctx(), int(ch)))
        if v == "auto":
            _lib.check(_lib.lib().chfsi_ctx_set_tiling(_lib.ctx(), 0, 0, 0))
        else:
            # "64x32d": two 8-warp groups per CTA; "128x32w8": 8 warps per group
            # "...g148": grid override (CTAs per launch)
            v0, _, gr = v.partition("g")
            vv, _, wp = v0.partition("w")
            dual = vv.endswith("d")
            bm, bn = (int(t) for t in vv.rstrip("d").split("x"))
            _lib.check(_lib.lib().chfsi_ctx_set_tiling(_lib.ctx(), bm, bn, int(gr) if gr else 0))
            if dual:
                _lib.check(_lib.lib().chfsi_ctx_set_step_groups(_lib.ctx(), 2))
            _lib.check(_lib.lib().chfsi_ctx_set_step_warps(_lib.ctx(), int(wp) if wp else 0))
        ms = timed(lambda: _filter_into(op, y, x, y, deg, win), reps) / deg
        fl = 8.0 * n * n * w
        print(json.dumps({"n": n, "w": w, "variant": v, "product": int(prod), "chains": int(ch), "k1_us": round(ms * 1e3, 2),
                          "k1_tflops": round(fl / ms / 1e9, 2),
                          "cublas_tflops": None if cub is None else round(cub, 2)}), flush=True)
    _lib.check(_lib.lib().chfsi_ctx_set_tiling(_lib.ctx(), 0, 0, 0))
