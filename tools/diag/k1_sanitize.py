"""Small K1 workload for compute-sanitizer (racecheck / synccheck / memcheck).

    compute-sanitizer --tool racecheck python tools/diag/k1_sanitize.py

Covers the TMA + mbarrier ring, both complex products (3M and 4M), one
and two tile groups per CTA, data-parallel tiles, stream-K splits with
owner folds (forced small grids), the conj flag and an in-place (aliased)
Yprev/Ynext step — each filter of degree 3 (three dependent K1 launches,
PDL between them), at sizes the instrumented run finishes in minutes.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200._lib import check, ctx, lib

CASES = [  # n, w, bm, grid, groups, warps, product, conj(column-major H)
    (256, 48, 64, 0, 1, 0, 3, False),
    (300, 33, 64, 37, 1, 0, 3, True),
    (300, 33, 64, 37, 2, 0, 4, False),
    (520, 40, 128, 13, 1, 0, 3, False),
    (200, 17, 64, 7, 1, 4, 3, True),
]


def main():
    torch.cuda.set_device(0)
    L = lib()
    rng = np.random.default_rng(0)
    for n, w, bm, grid, groups, warps, product, conj in CASES:
        g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        h = torch.from_numpy((g + g.conj().T) / 2).cuda()
        if conj:
            h = h.t().contiguous().t()  # column-major storage: the kernels read conj rows
        y = torch.from_numpy(rng.standard_normal((w, n)) + 1j * rng.standard_normal((w, n))).cuda().t()
        L.chfsi_set_complex_product(product)
        check(L.chfsi_ctx_set_tiling(ctx(), bm, 32, grid), "tiling")
        check(L.chfsi_ctx_set_step_groups(ctx(), groups), "groups")
        if warps:
            check(L.chfsi_ctx_set_step_warps(ctx(), warps), "warps")
        win = pkg.FilterWindow(a=-1.0, b=float(np.abs(g).sum(1).max()), scale_ref=-1.5)
        with pkg.array_output("torch"):
            a = pkg.chebyshev_filter(h, y, 3, win)
            b = pkg.chebyshev_filter(h, y, 3, win)
        torch.cuda.synchronize()
        same = bool(torch.equal(a, b))
        print(f"n={n} w={w} bm={bm} grid={grid} groups={groups} warps={warps} {product}M "
              f"conj={conj}: repeat-equal={same}", flush=True)
        check(L.chfsi_ctx_set_step_groups(ctx(), 1), "groups")
        check(L.chfsi_ctx_set_step_warps(ctx(), 0), "warps")
        check(L.chfsi_ctx_set_tiling(ctx(), 0, 0, 0), "tiling")
        if not same:
            sys.exit(1)
    L.chfsi_set_complex_product(3)
    print("k1_sanitize done", flush=True)


if __name__ == "__main__":
    main()
