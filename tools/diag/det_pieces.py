"""Bitwise run-to-run determinism of the dense pieces used by Cholesky-QR3."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, ctypes
import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import _lib
from paper_1206_3768_b200._device import fblock, to_fblock, ld_of
L = _lib.lib(); C = _lib.ctx(); dp = _lib.dptr
for (m, n) in [(2048, 160), (2048, 131), (2048, 97), (5000, 600)]:
    rng = np.random.default_rng(m + n)
    y = to_fblock(rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)))
    outs = {"gemm": [], "potrf": [], "trsm": [], "qr": []}
    for it in range(5):
        g = fblock(n, n)
        _lib.check(L.chfsi_gemm_z(C, b"C", b"N", n, n, m, 1.0, 0.0, dp(y), m, dp(y), m, 0.0, 0.0, dp(g), n))
        outs["gemm"].append(g.clone())
        info = ctypes.c_int()
        gg = g.clone()
        # upper Cholesky via the lower API on the conjugate: use chfsi_potrf_z (lower) on g
        _lib.check(L.chfsi_potrf_z(C, n, dp(gg), n, ctypes.byref(info)))
        outs["potrf"].append(gg.clone())
        yy = y.clone()
        _lib.check(L.chfsi_trsm_z(C, b"R", b"C", m, n, dp(gg), n, dp(yy), m))
        outs["trsm"].append(yy.clone())
        q = pkg.qr_orthonormalize(y)
        outs["qr"].append(q.clone())
    torch.cuda.synchronize()
    print(m, n, {k: all(torch.equal(v[0], x) for x in v[1:]) for k, v in outs.items()}, flush=True)
