"""Latency of the Rayleigh-Ritz w x w eigensolvers in isolation: the
near-diagonal Jacobi/Newton-Schulz path (chfsi_heev_rr_z with a tolerance)
vs cuSOLVER zheevd, for G = D + E with off-diagonal/gap ratio r.

    python tools/diag/rr_eig_bench.py
"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_1206_3768_b200._device import fblock
from paper_1206_3768_b200._lib import check, ctx, dptr, lib


def make_g(w, r, rng):
    d = np.sort(rng.uniform(-1, 9, w))
    gap = np.min(np.diff(d))
    e = (rng.standard_normal((w, w)) + 1j * rng.standard_normal((w, w)))
    e = (e + e.conj().T) / 2
    np.fill_diagonal(e, 0)
    e *= r * gap / np.abs(e).max()
    return np.diag(d).astype(complex) + e


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    L = lib()
    for w in (48, 100, 160):
        for r in (1e-6, 1e-3, 1e-1, 0.4):
            g = make_g(w, r, rng)
            g0 = fblock(w, w)
            g0.copy_(torch.from_numpy(g))
            a = fblock(w, w)
            wd = torch.empty(w, dtype=torch.float64, device="cuda")
            used = ctypes.c_int()
            res = {}
            for name, tol in (("nd", 1e-13), ("zheevd", 0.0)):
                times = []
                for rep in range(12):
                    a.copy_(g0)
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    check(L.chfsi_heev_rr_z(ctx(), w, dptr(a), w, dptr(wd), tol, ctypes.byref(used)),
                          "heev_rr")
                    torch.cuda.synchronize()
                    if rep >= 2:
                        times.append(time.perf_counter() - t0)
                res[name] = (1e6 * float(np.median(times)), used.value)
            print(f"w={w:4d} r={r:7.0e}  near-diag {res['nd'][0]:8.1f} us (used={res['nd'][1]})   "
                  f"zheevd {res['zheevd'][0]:8.1f} us", flush=True)


if __name__ == "__main__":
    main()
