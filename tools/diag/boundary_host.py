"""Host time at the problem boundaries of a C2 sequence (device idle there):
driver marks (CHFSI_DRIVER_TRACE) and chfsi_solve's own host phases.

    python tools/diag/boundary_host.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ["CHFSI_DRIVER_TRACE"] = "1"

import numpy as np
import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import harness
from paper_1206_3768_b200.harness import default_config, solve_sequence

torch.cuda.set_device(0)
cfg_b = pkg.BASELINE_CONFIGS["C2"]
cfg = default_config(cfg_b)
pencils = [pkg.EigenPencil(a=x, b=y, label=lab)
           for lab, x, y in pkg.iter_baseline_sequence(cfg_b.n, cfg_b.length, seed=0, device=0)]
for _ in range(4):
    solve_sequence(pencils, cfg, seed=0)
torch.cuda.synchronize()
acc = {}
reps = 5
for _ in range(reps):
    harness.DRIVER_TRACE.clear()
    res = solve_sequence(pencils, cfg, seed=0)
    torch.cuda.synchronize()
    tr = list(harness.DRIVER_TRACE)
    for (a, ta), (b, tb) in zip(tr[:-1], tr[1:]):
        key = f"{a} -> {b}"
        acc.setdefault(key, []).append((tb - ta) * 1e3)
    for r in res[1:]:
        for k, v in r.report.host_phases.items():
            acc.setdefault(f"solve.{k}", []).append(v * 1e3)
    res = None
for k, v in acc.items():
    print(f"{k:42s} n={len(v) // reps:3d}/seq  mean {np.mean(v):8.3f} ms  total/seq {np.sum(v) / reps:8.2f} ms")
