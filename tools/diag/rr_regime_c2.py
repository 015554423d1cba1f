import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_1206_3768_b200 as pkg
from paper_1206_3768_b200.harness import default_config, solve_sequence
cfg_b = pkg.BASELINE_CONFIGS["C2"]
seq = list(pkg.iter_baseline_sequence(cfg_b.n, cfg_b.length, seed=0, device=0))
pencils = [pkg.EigenPencil(a=x, b=y, label=l) for l, x, y in seq]
res = solve_sequence(pencils, default_config(cfg_b), seed=0)
for r in res: print("problem", r.label, "loops", r.report.inner_loops, "fast", r.report.rr_fast_eigs, file=sys.stderr)
