"""Run-to-run / driver-mode determinism of a C1 sequence in one process:
threaded, inline and serial drivers, each twice, after a warm-up that
leaves the solver stream's caches populated. Prints which pairs differ.

    python tools/diag/det_streams.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1206_3768_b200 as pkg


def run(seq, cfg, mode):
    if mode == "inline":
        os.environ["CHFSI_SIDE_WORKER"] = "0"
    try:
        return pkg.solve_sequence(seq, cfg, seed=0, overlap=(mode != "serial"))
    finally:
        os.environ.pop("CHFSI_SIDE_WORKER", None)


def main():
    torch.cuda.set_device(0)
    pkg.set_array_output("torch")
    cfg_b = pkg.BASELINE_CONFIGS["C1"]
    cfg = pkg.ChfsiConfig(nev=cfg_b.nev, nex=cfg_b.nex, deg=cfg_b.deg, tol=cfg_b.tol)
    seq = list(pkg.iter_baseline_sequence(cfg_b.n, 4, seed=0))
    # warm-up: other shapes and modes first (as the test file does)
    h = np.random.default_rng(1).standard_normal((300, 300)) + 0j
    pkg.chfsi_solve(h + h.T, pkg.ChfsiConfig(nev=8, blk=24, deg=10), rng=3)
    runs = {}
    for mode in ("threaded", "inline", "serial", "threaded", "inline", "serial"):
        res = run(seq, cfg, mode)
        runs.setdefault(mode, []).append(res)
    names = [(m, i) for m in runs for i in range(len(runs[m]))]
    base = runs["serial"][0]
    for m, i in names:
        r = runs[m][i]
        dv = max(float(np.abs(a.values - b.values).max()) for a, b in zip(base, r))
        dx = max(float((a.solution.vectors - b.solution.vectors).abs().max()) for a, b in zip(base, r))
        same = all(np.array_equal(a.values, b.values) and torch.equal(a.solution.vectors,
                                                                    b.solution.vectors)
                   for a, b in zip(base, r))
        print(f"{m}#{i} vs serial#0: bitwise={same} max|dvalues|={dv:.3e} max|dx|={dx:.3e}",
              flush=True)


if __name__ == "__main__":
    main()
