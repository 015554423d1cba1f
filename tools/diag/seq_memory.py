"""Device memory in use after each problem of a C1 sequence (leak check of
the sequence driver), per driver variant given by the environment."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch

import paper_1206_3768_b200 as pkg
import paper_1206_3768_b200.harness as hs

cfg_b = pkg.BASELINE_CONFIGS["C1"]
cfg = pkg.ChfsiConfig(nev=cfg_b.nev, nex=cfg_b.nex, deg=cfg_b.deg, tol=cfg_b.tol)
dev = torch.device("cuda", 0)
seq = [pkg.EigenPencil(a=torch.from_numpy(a).to(dev), b=torch.from_numpy(b).to(dev), label=lab)
       for lab, a, b in pkg.iter_baseline_sequence(cfg_b.n, 6, seed=0)]
for variant in ("default", "nogc_off"):
    if variant == "nogc_off":
        hs.gc.disable = lambda: None  # keep collections on inside the call
    pkg.solve_sequence(seq, cfg, seed=0)
    used = []
    pkg.solve_sequence(seq, cfg, seed=0,
                       on_problem=lambda r: used.append(torch.cuda.memory_allocated(dev) >> 10))
    print(os.environ.get("TAG", ""), variant, used, flush=True)
