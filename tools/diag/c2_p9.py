"""Diagnose C2 problem 9 warm (harness protocol) under forced K1 tilings."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import _lib
cfg_b = pkg.BASELINE_CONFIGS["C2"]
cfg = pkg.ChfsiConfig(nev=cfg_b.nev, nex=cfg_b.nex, deg=cfg_b.deg, tol=cfg_b.tol)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, 9, seed=0))
sp8 = pkg.to_standard(pkg.EigenPencil(a=seq[7][1], b=seq[7][2], label=8))
dv, dvec = pkg.hermitian_eig(sp8.h)
sp9 = pkg.to_standard(pkg.EigenPencil(a=seq[8][1], b=seq[8][2], label=9))
guess = pkg.ChfsiGuess(vectors=dvec[:, :cfg_b.blk], lambda1=float(dv[0]), lambda_blk_plus_1=float(dv[cfg_b.blk]))
for til in [(0,0,0), (64,32,0), (128,32,0), (32,32,0), (64,16,0), (64,64,0), (64,32,0), (64,32,7)]:
    _lib.check(_lib.lib().chfsi_ctx_set_tiling(_lib.ctx(), *til))
    sol, rep = pkg.chfsi_solve(sp9.h, cfg, guess=guess, rng=np.random.default_rng((0, 9, 1)))
    print(til, rep.inner_loops, rep.locked_per_loop, sol.values[:3])
