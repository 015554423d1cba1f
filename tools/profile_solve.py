"""One warm problem (chained from problem 1) between cudaProfilerStart/Stop,
for `ncu --profile-from-start off` launch lists.

    python tools/profile_solve.py [--config C2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200.harness import default_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
a = ap.parse_args()
cfg_b = pkg.BASELINE_CONFIGS[a.config]
cfg = default_config(cfg_b)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, 2, seed=0))
res = pkg.solve_sequence(seq[:1], cfg)
r1 = res[0]
guess = pkg.ChfsiGuess(vectors=r1.report.tail_vectors, lambda1=float(r1.values[0]),
                       lambda_blk_plus_1=float(r1.report.lambda_blk_plus_1))
pencil = pkg.EigenPencil(a=seq[1][1], b=seq[1][2], label=2)
torch.cuda.synchronize()
torch.cuda.profiler.start()
sp = pkg.to_standard(pencil)
sol, rep = pkg.chfsi_solve(sp.h, cfg, guess=guess, rng=np.random.default_rng((0, 2, 1)))
x = pkg.back_transform(sp.cholesky_factor, sol)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("loops", rep.inner_loops, "filter ms", rep.t_filter * 1e3, "ortho", rep.t_ortho * 1e3,
      "rr", rep.t_rr * 1e3, "lanczos", rep.t_lanczos * 1e3)
