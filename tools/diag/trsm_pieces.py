"""Pieces of the block triangular solves at n = 2048 (CUDA events): cuBLAS
ZTRSM on an nb-row diagonal block with m right-hand sides, and the K1 update."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import ctypes

import torch

from paper_1206_3768_b200 import _lib
from paper_1206_3768_b200._device import fblock

L = _lib.lib()
P = lambda t, off=0: ctypes.c_void_p(t.data_ptr() + off)  # noqa: E731
c = _lib.ctx()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


n = 2048
g = torch.randn(n, n, dtype=torch.complex128, device="cuda")
b = torch.eye(n, dtype=torch.complex128, device="cuda") + g @ g.conj().T / (4 * n)
lt = torch.linalg.cholesky(b)  # lower
lf = lt.t().contiguous().t()   # column-major
for nb in (128, 256, 512):
    for m in (128, 2048):
        r = fblock(n, m)
        r.copy_(torch.randn(n, m, dtype=torch.complex128, device="cuda"))
        us = timed(lambda: _lib.check(L.chfsi_trsm_z(c, b"L", b"N", nb, m, P(lf), n, P(r), n)))
        print(f"ztrsm diag nb={nb} m={m}: {us:.1f} us")
        us = timed(lambda: _lib.check(L.chfsi_cheb_step_rows_z(
            c, n // 2, nb, m, P(lf, 16 * (n // 2) * n), n, 1, P(r), n, 0, 0, P(r, 16 * (n // 2)), n,
            P(r, 16 * (n // 2)), n, P(r, 16 * (n // 2)), n, -1.0, 0.0, -1.0)))
        print(f"k1 update rows={nb} k={n // 2} m={m}: {us:.1f} us")

# whole reductions at larger n: K1 block substitutions vs the ZTRSM path
import time as _t

from paper_1206_3768_b200.reduction import stage_standard

import paper_1206_3768_b200 as pkg

for n in (2048, 5000, 12000):
    g = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    a = (g + g.conj().T) / 2
    b = torch.eye(n, dtype=torch.complex128, device="cuda") + g @ g.conj().T / (4 * n)
    del g
    for name, fn in (("k1", lambda: stage_standard(a, b, 1, check_hermitian=False)),
                     ("ztrsm", lambda: pkg.to_standard(pkg.EigenPencil(a=a, b=b, validate=False)))):
        fn()
        torch.cuda.synchronize()
        t = _t.perf_counter()
        reps = 3 if n < 10000 else 1
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        print(f"reduce n={n} {name}: {(_t.perf_counter() - t) / reps * 1e3:.1f} ms")
    del a, b
    torch.cuda.empty_cache()
