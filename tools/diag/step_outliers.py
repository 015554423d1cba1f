"""Per-step C2 sequence times with the caching allocator's device-malloc
count and the GC state around each step (what makes an occasional step
slow?).

    python tools/diag/step_outliers.py [--steps 20]
"""
import argparse
import gc
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

os.environ.setdefault("CHFSI_DRIVER_TRACE", "1")

import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import harness
from paper_1206_3768_b200.harness import default_config, solve_sequence

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
torch.cuda.set_device(0)
cfg_b = pkg.BASELINE_CONFIGS["C2"]
cfg = default_config(cfg_b)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, cfg_b.length, seed=0))
pencils = [pkg.EigenPencil(a=torch.from_numpy(x).cuda(), b=torch.from_numpy(y).cuda(), label=l)
           for l, x, y in seq]
for _ in range(3):
    solve_sequence(pencils, cfg, seed=0)
gc.collect()
gc.freeze()
torch.cuda.synchronize()
res = None
for i in range(a.steps):
    st0 = torch.cuda.memory_stats()
    c0 = gc.get_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    res = None
    harness.DRIVER_TRACE.clear()
    res = solve_sequence(pencils, cfg, seed=0)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    st1 = torch.cuda.memory_stats()
    per = [round(r.t_solve * 1e3, 1) for r in res]
    red = [round(r.t_reduce * 1e3, 1) for r in res]
    stg = [round(r.extra.get("t_stage_next", 0.0) * 1e3, 1) for r in res]
    tb = [round(r.t_back * 1e3, 1) for r in res]
    solves = sum(r.t_solve for r in res) * 1e3
    print(f"step {i:2d}: dev {e0.elapsed_time(e1):7.1f} ms wall {wall * 1e3:7.1f} ms "
          f"cudaMalloc +{st1['num_device_alloc'] - st0['num_device_alloc']} "
          f"free +{st1['num_device_free'] - st0['num_device_free']} "
          f"retries +{st1['num_alloc_retries'] - st0['num_alloc_retries']} gc {c0} "
          f"slowest problem {max(per)} ms (#{per.index(max(per)) + 1}) solves {solves:.1f} "
          f"wait-staged {red} stage-submit {stg} back {tb}", flush=True)
    tr = harness.DRIVER_TRACE
    if tr and e0.elapsed_time(e1) > 300.0:
        gaps = [(tr[k][0] + "->" + tr[k + 1][0], round((tr[k + 1][1] - tr[k][1]) * 1e3, 2))
                for k in range(len(tr) - 1)]
        big = sorted(gaps, key=lambda g: -g[1])[:6]
        print("    host timeline: enter->exit %.1f ms, largest gaps %s" %
              ((tr[-1][1] - tr[0][1]) * 1e3, big), flush=True)
