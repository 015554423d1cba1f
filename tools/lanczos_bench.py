"""Cold-start Lanczos (K2) time at the BASELINE shapes vs its HBM bound.

    python tools/lanczos_bench.py [--shapes 2048x204,5000x500,12000x1200]
Bound: k GEMVs stream H (16 n^2 bytes each) at the measured HBM bandwidth.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_1206_3768_b200._device import Operator
from paper_1206_3768_b200.chfsi import _lanczos_estimates

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="2048x204,5000x500,12000x1200")
a = ap.parse_args()
hbm = 7.0e12
try:
    mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    for k, v in mp.items():
        if "hbm" in k.lower() and isinstance(v, (int, float)):
            hbm = float(v) * (1e9 if v < 1e5 else 1.0)
            break
except (OSError, ValueError):
    pass
for shape in a.shapes.split(","):
    n, k = (int(x) for x in shape.split("x"))
    g = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    h = (g + g.conj().T) / 2
    del g
    op = Operator(h)
    _lanczos_estimates(op, min(k, 20), np.random.default_rng(0))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ritz, beta, steps = _lanczos_estimates(op, k, np.random.default_rng(1))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    bound = steps * 16.0 * n * n / hbm
    print(json.dumps({"n": n, "k": k, "steps": steps, "ms": round(dt * 1e3, 2),
                      "ms_per_step": round(dt * 1e3 / steps, 4),
                      "hbm_bound_ms": round(bound * 1e3, 2), "frac_of_bound": round(bound / dt, 3)}),
          flush=True)
    del h, op
    torch.cuda.empty_cache()
