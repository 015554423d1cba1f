"""Is one solve bitwise the same on the default stream, a fresh stream and a
highest-priority stream? (C1 problem 1, cold start.) Then the pieces:
Lanczos, one filter, QR, one Rayleigh-Ritz on each stream.

    python tools/diag/det_priority.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1206_3768_b200 as pkg


def main():
    torch.cuda.set_device(0)
    pkg.set_array_output("torch")
    cfg_b = pkg.BASELINE_CONFIGS["C1"]
    cfg = pkg.ChfsiConfig(nev=cfg_b.nev, nex=cfg_b.nex, deg=cfg_b.deg, tol=cfg_b.tol)
    lab, a, b = next(iter(pkg.iter_baseline_sequence(cfg_b.n, 1, seed=0)))
    sp = pkg.to_standard(pkg.EigenPencil(a=torch.from_numpy(a).cuda(), b=torch.from_numpy(b).cuda()))
    h = sp.h.clone()
    torch.cuda.synchronize()
    streams = {"default": torch.cuda.current_stream(), "fresh": torch.cuda.Stream(),
               "high": torch.cuda.Stream(priority=-100), "low": torch.cuda.Stream(priority=0)}
    out = {}
    for name, st in streams.items():
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            sol, rep = pkg.chfsi_solve(h, cfg, rng=np.random.default_rng((0, 1, 0)))
            win = pkg.FilterWindow(a=0.5, b=9.5, scale_ref=-1.0)
            g = torch.Generator(device="cpu").manual_seed(5)
            y = torch.randn((h.shape[0], 48), dtype=torch.complex128, generator=g).cuda()
            f = pkg.chebyshev_filter(h, y.t().contiguous().t(), 12, win)
            q = pkg.qr_orthonormalize(f)
            ritz, rot = pkg.rayleigh_ritz(h, q)
            lb = pkg.lanczos_upper_bound(h, 60, rng=3)
        st.synchronize()
        out[name] = (sol.values, sol.vectors.clone(), f.clone(), q.clone(), ritz, rot.clone(), lb)
    ref = out["default"]
    for name, r in out.items():
        flags = [np.array_equal(ref[0], r[0]), torch.equal(ref[1], r[1]), torch.equal(ref[2], r[2]),
                 torch.equal(ref[3], r[3]), np.array_equal(ref[4], r[4]), torch.equal(ref[5], r[5]),
                 ref[6] == r[6]]
        print(name, "values,vectors,filter,qr,ritz,rot,lanczos bitwise:", flags,
              f"max|dvalues|={float(np.abs(ref[0] - r[0]).max()):.2e}", flush=True)


if __name__ == "__main__":
    main()
