"""Run the C2 chained sequence repeatedly; counts must be identical run to run."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import _lib
from paper_1206_3768_b200.harness import default_config
cfg_b = pkg.BASELINE_CONFIGS["C2"]
cfg = default_config(cfg_b)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, cfg_b.length, seed=0))
dev = torch.device("cuda", 0)
pencils = [pkg.EigenPencil(a=torch.from_numpy(a).to(dev), b=torch.from_numpy(b).to(dev), label=l) for l, a, b in seq]
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
_lib.check(_lib.lib().chfsi_ctx_set_qr_mode(_lib.ctx(), mode))
ref = None
for it in range(6):
    res = pkg.solve_sequence(pencils, cfg, mode="chained")
    loops = [r.report.inner_loops for r in res]
    vals = np.concatenate([r.values for r in res])
    same = ref is not None and np.array_equal(vals, ref)
    print("mode", mode, "run", it, loops, "bitwise-equal-to-run0:", same, flush=True)
    if ref is None:
        ref = vals
