"""Host-side outliers of the chained C2 sequence: per problem wall time and
its host phases, over several repetitions.

    python tools/diag/outliers.py [--reps 6]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200.harness import default_config, solve_sequence

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=6)
ap.add_argument("--config", default="C2")
ap.add_argument("--no-overlap", action="store_true")
ap.add_argument("--no-gc", action="store_true")
a = ap.parse_args()
import gc

gc_log = []
if a.no_gc:
    gc.disable()
else:
    _gc_t = {}

    def _gc_cb(phase, info):
        if phase == "start":
            _gc_t["t"] = time.perf_counter()
        else:
            gc_log.append((info.get("generation"), (time.perf_counter() - _gc_t.get("t", 0)) * 1e3))

    gc.callbacks.append(_gc_cb)
cfg_b = pkg.BASELINE_CONFIGS[a.config]
cfg = default_config(cfg_b)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, cfg_b.length, seed=0))
dev = torch.device("cuda", 0)
pencils = [pkg.EigenPencil(a=torch.from_numpy(x).to(dev), b=torch.from_numpy(y).to(dev), label=lab)
           for lab, x, y in seq]
runs = []
mallocs = []
for r in range(a.reps + 2):
    m0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    t0 = time.perf_counter()
    res = solve_sequence(pencils, cfg, seed=0, overlap=not a.no_overlap)
    torch.cuda.synchronize()
    runs.append((time.perf_counter() - t0, res))
    st = torch.cuda.memory_stats()
    mallocs.append((st.get("num_device_alloc", 0) - m0, st.get("num_device_free"),
                    st.get("num_alloc_retries"), st.get("num_sync_all_streams"),
                    round(st.get("reserved_bytes.all.current", 0) / 2**20)))
mallocs = mallocs[2:]
runs = runs[2:]
best = {}
for _, res in runs:
    for p in res:
        best[p.label] = min(best.get(p.label, 1e9), p.t_solve)
big = [g for g in gc_log if g[1] > 2.0]
print(f"gc passes {len(gc_log)}, >2 ms: {len(big)}, max {max([g[1] for g in gc_log] or [0]):.1f} ms")
for i, (wall, res) in enumerate(runs):
    print(f"run {i}: wall {wall * 1e3:.1f} ms  cudaMalloc calls {mallocs[i]}")
    for p in res:
        if p.t_solve > 1.3 * best[p.label] + 2e-3:
            hp = {k: round(v * 1e3, 1) for k, v in p.report.host_phases.items()}
            dv = round(1e3 * (p.report.t_filter + p.report.t_ortho + p.report.t_rr), 1)
            print(f"  outlier label {p.label}: t_solve {p.t_solve * 1e3:.1f} (best "
                  f"{best[p.label] * 1e3:.1f}) reduce {p.t_reduce * 1e3:.1f} back {p.t_back * 1e3:.1f} "
                  f"host {hp} loop-device {dv}")
