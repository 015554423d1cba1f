"""Bitwise determinism of qr_orthonormalize (mode 0) over widths and conditioning."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import _lib
from paper_1206_3768_b200._device import to_fblock
m = 2048
rng = np.random.default_rng(0)
bad = []
for n in range(30, 161, 3):
    for scale in (0, 6, 10):
        y = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        y = y * np.logspace(0, -scale, n)
        yd = to_fblock(y)
        qs = [pkg.qr_orthonormalize(yd) for _ in range(4)]
        if not all(torch.equal(qs[0], q) for q in qs[1:]):
            bad.append((n, scale))
print("nondeterministic qr (n, scale):", bad)
