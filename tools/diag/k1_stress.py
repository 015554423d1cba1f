"""Stress K1 for rare races: repeat the same filter many times, report mismatching tiles."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200._device import to_fblock, Operator
n = 2048
rng = np.random.default_rng(0)
g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
h = torch.from_numpy((g + g.conj().T) / 2).cuda()
hcol = h.t().contiguous().t()
win = pkg.FilterWindow(a=-1.0, b=30.0, scale_ref=-40.0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for w in (160, 149, 131, 97, 64, 40):
    y = to_fblock(rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w)))
    for hh in (h, hcol):
        ref = pkg.chebyshev_filter(hh, y, 4, win).clone()
        bad = 0
        for it in range(reps):
            out = pkg.chebyshev_filter(hh, y, 4, win)
            if not torch.equal(out, ref):
                bad += 1
                d = (out - ref).abs()
                rows = torch.nonzero(d.amax(dim=1) > 0).flatten()
                cols = torch.nonzero(d.amax(dim=0) > 0).flatten()
                print(f"w={w} conj={hh is hcol} rep {it}: rows {rows.min().item()}..{rows.max().item()} ({rows.numel()}),"
                      f" cols {cols.min().item()}..{cols.max().item()} ({cols.numel()}), max {d.max().item():.3e}", flush=True)
        print(f"w={w} conj={hh is hcol}: {bad}/{reps} mismatches", flush=True)
