"""Does earlier work on the same libchfsi context change a later result?
Runs the C1 sequence serially on the caller's stream, then one 'polluting'
operation at n = 2048 on the same stream, then the C1 sequence again, and
compares bit for bit.

    python tools/diag/det_pollution.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1206_3768_b200 as pkg


def c1(seq, cfg):
    return pkg.solve_sequence(seq, cfg, seed=0, overlap=False)


def same(r1, r2):
    return all(np.array_equal(a.values, b.values) and torch.equal(a.solution.vectors, b.solution.vectors)
               for a, b in zip(r1, r2))


def main():
    torch.cuda.set_device(0)
    pkg.set_array_output("torch")
    cfg_b = pkg.BASELINE_CONFIGS["C1"]
    cfg = pkg.ChfsiConfig(nev=cfg_b.nev, nex=cfg_b.nex, deg=cfg_b.deg, tol=cfg_b.tol)
    seq = list(pkg.iter_baseline_sequence(cfg_b.n, 3, seed=0))
    base = c1(seq, cfg)
    rng = np.random.default_rng(0)
    g = rng.standard_normal((2048, 2048)) + 1j * rng.standard_normal((2048, 2048))
    big = torch.from_numpy((g + g.conj().T) / 2).cuda()
    c2seq = list(pkg.iter_baseline_sequence(2048, 1, seed=0))
    ops = {
        "hermitian_eig(2048)": lambda: pkg.hermitian_eig(big),
        "to_standard(2048)": lambda: pkg.to_standard(pkg.EigenPencil(a=c2seq[0][1], b=c2seq[0][2])),
        "chfsi_solve(2048)": lambda: pkg.chfsi_solve(big, pkg.ChfsiConfig(nev=128, nex=32, deg=16),
                                                     rng=1),
        "qr(2048x160)": lambda: pkg.qr_orthonormalize(torch.randn(2048, 160, dtype=torch.complex128,
                                                                  device="cuda")),
    }
    for name, op in ops.items():
        op()
        torch.cuda.synchronize()
        r = c1(seq, cfg)
        dv = max(float(np.abs(a.values - b.values).max()) for a, b in zip(base, r))
        print(f"after {name}: bitwise={same(base, r)} max|dvalues|={dv:.2e}", flush=True)


if __name__ == "__main__":
    main()
