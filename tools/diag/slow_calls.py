"""Find host-side calls that take > 5 ms during repeated C2 sequences
(torch profiler, CPU + CUDA runtime activities).

    python tools/diag/slow_calls.py [--reps 8]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch
from torch.profiler import ProfilerActivity, profile

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200.harness import default_config, solve_sequence

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=8)
a = ap.parse_args()
cfg_b = pkg.BASELINE_CONFIGS["C2"]
cfg = default_config(cfg_b)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, cfg_b.length, seed=0))
dev = torch.device("cuda", 0)
pencils = [pkg.EigenPencil(a=torch.from_numpy(x).to(dev), b=torch.from_numpy(y).to(dev), label=lab)
           for lab, x, y in seq]
for _ in range(2):
    solve_sequence(pencils, cfg, seed=0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        solve_sequence(pencils, cfg, seed=0)
    torch.cuda.synchronize()
slow = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CPU:
        d = (e.time_range.end - e.time_range.start) / 1e3
        if d > 5.0:
            slow.append((d, e.name, e.time_range.start))
slow.sort(key=lambda x: -x[0])
print(f"{len(slow)} host calls > 5 ms")
for d, name, t in slow[:40]:
    print(f"{d:9.2f} ms  {name[:100]}")
