"""C2 chained problems 1..6 under QR mode 0 (Cholesky-QR3) vs 1 (Householder)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import _lib
from paper_1206_3768_b200.harness import default_config
cfg_b = pkg.BASELINE_CONFIGS["C2"]
cfg = default_config(cfg_b)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, 7, seed=0))
for mode in (1, 0, 0):
    _lib.check(_lib.lib().chfsi_ctx_set_qr_mode(_lib.ctx(), mode))
    res = pkg.solve_sequence(seq, cfg, mode="chained")
    print("mode", mode, [(r.report.inner_loops, r.report.locked_per_loop) for r in res][4:])
