"""Near-diagonal RR eigensolver regime per pass over one chained sequence
(run with CHFSI_RR_DEBUG=1: the library prints rmax/emax per step)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200.harness import default_config, solve_sequence

cfg_b = pkg.BASELINE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
seq = list(pkg.iter_baseline_sequence(cfg_b.n, int(sys.argv[2]) if len(sys.argv) > 2 else 2, seed=0))
dev = torch.device("cuda", 0)
pencils = [pkg.EigenPencil(a=torch.from_numpy(x).to(dev), b=torch.from_numpy(y).to(dev), label=lab)
           for lab, x, y in seq]
res = solve_sequence(pencils, default_config(cfg_b), seed=0, overlap=False)
torch.cuda.synchronize()
for r in res:
    print("problem", r.label, "loops", r.report.inner_loops, "fast", r.report.rr_fast_eigs,
          "locked", r.report.locked_per_loop, file=sys.stderr)
