"""Bitwise determinism of the Gram ZGEMM over the panel widths the solve visits."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, ctypes
import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import _lib
from paper_1206_3768_b200._device import fblock, to_fblock
L = _lib.lib(); C = _lib.ctx(); dp = _lib.dptr
m = 2048
rng = np.random.default_rng(0)
base = to_fblock(rng.standard_normal((m, 200)) + 1j * rng.standard_normal((m, 200)))
bad = []
for off in (0, 3, 17):
    for n in range(30, 161, 1):
        y = base[:, off:off + n]
        res = []
        for it in range(4):
            g = fblock(n, n)
            _lib.check(L.chfsi_gemm_z(C, b"C", b"N", n, n, m, 1.0, 0.0, dp(y), m, dp(y), m, 0.0, 0.0, dp(g), n))
            res.append(g.clone())
        if not all(torch.equal(res[0], r) for r in res[1:]):
            bad.append((off, n))
print("nondeterministic (offset, n):", bad[:40], len(bad))
# the potrf/trsm pieces on a fixed Gram
bad2 = []
for n in range(30, 161, 7):
    y = base[:, :n].clone()
    g = fblock(n, n)
    _lib.check(L.chfsi_gemm_z(C, b"C", b"N", n, n, m, 1.0, 0.0, dp(y), m, dp(y), m, 0.0, 0.0, dp(g), n))
    rs = []
    for it in range(4):
        gg = g.clone(); info = ctypes.c_int()
        _lib.check(L.chfsi_potrf_z(C, n, dp(gg), n, ctypes.byref(info)))
        yy = y.clone()
        _lib.check(L.chfsi_trsm_z(C, b"R", b"C", m, n, dp(gg), n, dp(yy), m))
        rs.append((gg, yy))
    if not all(torch.equal(rs[0][0], r[0]) and torch.equal(rs[0][1], r[1]) for r in rs[1:]):
        bad2.append(n)
print("potrf/trsm nondeterministic n:", bad2)
