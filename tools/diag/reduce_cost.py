"""How much of the C2 sequence time the (side-stream) reduction to standard
form really costs: solve_sequence vs the same chained loop over problems
reduced ahead of time (outside the timed region).

    python tools/diag/reduce_cost.py [--config C2] [--reps 3]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200.harness import default_config, solve_sequence
from paper_1206_3768_b200.reduction import back_transform, stage_standard

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg_b = pkg.BASELINE_CONFIGS[a.config]
cfg = default_config(cfg_b)
dev = torch.device("cuda", 0)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, cfg_b.length, seed=0))
pencils = [pkg.EigenPencil(a=torch.from_numpy(x).to(dev), b=torch.from_numpy(y).to(dev), label=lab)
           for lab, x, y in seq]


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3


def pipeline():
    solve_sequence(pencils, cfg, seed=0)


staged = [stage_standard(p.a, p.b, p.label, check_hermitian=False)[1] for p in pencils]
torch.cuda.synchronize()


def prereduced():
    guess = None
    for p, sp in zip(pencils, staged):
        rng = np.random.default_rng((0, p.label, 0 if guess is None else 1))
        sol, rep = pkg.chfsi_solve(sp.h, cfg, guess=guess, rng=rng, label=p.label)
        back_transform(sp.cholesky_factor, sol)
        guess = pkg.ChfsiGuess(vectors=rep.tail_vectors, lambda1=float(sol.values[0]),
                               lambda_blk_plus_1=float(rep.lambda_blk_plus_1))


def reduce_only():
    for p in pencils:
        stage_standard(p.a, p.b, p.label, check_hermitian=False)


for name, fn in (("pipeline", pipeline), ("prereduced", prereduced), ("reduce_only", reduce_only)):
    fn()
    ts = [timed(fn) for _ in range(a.reps)]
    print(f"{name:12s} ms: {[round(t, 1) for t in ts]}  min {min(ts):.1f}")
