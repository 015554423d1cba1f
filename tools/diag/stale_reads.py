"""Do any cached device buffers get read before they are written? Poison
the reduction scratch and the solver workspace with NaN (then with zeros)
and compare the results bit for bit with a clean run.

    python tools/diag/stale_reads.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import chfsi as chfsi_mod
from paper_1206_3768_b200 import reduction


def poison(fill):
    for key, w in list(reduction._STAGING_WORK.items()):
        w.fill_(fill)
    for key, ws in list(chfsi_mod._WORKSPACES.items()):
        bufs = ws[0] + list(ws[1:-3])
        for b in bufs:
            b.fill_(fill)
        ws[-3].fill_(fill.real if isinstance(fill, complex) else fill)
        ws[-2].fill_(fill.real if isinstance(fill, complex) else fill)
    torch.cuda.synchronize()


def main():
    torch.cuda.set_device(0)
    pkg.set_array_output("torch")
    cfg_b = pkg.BASELINE_CONFIGS["C1"]
    cfg = pkg.ChfsiConfig(nev=cfg_b.nev, nex=cfg_b.nex, deg=cfg_b.deg, tol=cfg_b.tol)
    seq = list(pkg.iter_baseline_sequence(cfg_b.n, 4, seed=0))
    for overlap in (True, False):
        ref = pkg.solve_sequence(seq, cfg, seed=0, overlap=overlap)
        for fill in (complex(float("nan"), float("nan")), complex(1e300, -1e300), 0j):
            poison(fill)
            res = pkg.solve_sequence(seq, cfg, seed=0, overlap=overlap)
            same = all(np.array_equal(a.values, b.values) and torch.equal(a.solution.vectors,
                                                                        b.solution.vectors)
                       for a, b in zip(ref, res))
            finite = all(np.isfinite(b.values).all() for b in res)
            print(f"overlap={overlap} poison={fill}: bitwise={same} finite={finite}", flush=True)


if __name__ == "__main__":
    main()
