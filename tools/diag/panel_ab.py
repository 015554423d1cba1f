"""A/B of the Cholesky-QR2 panel kernels (panel_kernels.cu) vs the cuBLAS
chains: device time of chfsi_qr_orthonormalize_z at the C2 panel shapes,
then the C2 sequence with both settings.

    python tools/diag/panel_ab.py [--seq-steps 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import _lib as L, linalg
from paper_1206_3768_b200.harness import default_config, solve_sequence

ap = argparse.ArgumentParser()
ap.add_argument("--seq-steps", type=int, default=5)
a = ap.parse_args()
torch.cuda.set_device(0)
lib = L.lib()
rng = np.random.default_rng(0)
for m, n in [(2048, 160), (2048, 100), (2048, 48), (512, 48)]:
    y0 = torch.from_numpy((rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m)))
                          * np.logspace(0, -1.5, n)[:, None]).cuda().t()  # column-major m x n
    row = {}
    for on in (0, 1):
        lib.chfsi_set_panel_kernels(on)
        ts = []
        for rep in range(12):
            y = y0.clone(memory_format=torch.preserve_format)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            linalg.qr_orthonormalize_inplace(y)
            e1.record()
            torch.cuda.synchronize()
            if rep >= 2:
                ts.append(e0.elapsed_time(e1) * 1e3)
        row[on] = sorted(ts)[len(ts) // 2]
    print(f"qr {m} x {n}: library {row[0]:.1f} us, panel kernels {row[1]:.1f} us (incl. the host sync of the test)",
          flush=True)

cfg_b = pkg.BASELINE_CONFIGS["C2"]
cfg = default_config(cfg_b)
pencils = [pkg.EigenPencil(a=x, b=y, label=lab)
           for lab, x, y in pkg.iter_baseline_sequence(cfg_b.n, cfg_b.length, seed=0, device=0)]
for rnd in range(2):
    for on in (1, 0):
        lib.chfsi_set_panel_kernels(on)
        for _ in range(3):
            solve_sequence(pencils, cfg, seed=0)
        torch.cuda.synchronize()
        ts, ortho, loops = [], 0.0, None
        for _ in range(a.seq_steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = solve_sequence(pencils, cfg, seed=0)
            e1.record()
            torch.cuda.synchronize()
            ts.append(round(e0.elapsed_time(e1), 1))
            ortho = sum(r.report.t_ortho for r in res) * 1e3
            loops = [r.report.inner_loops for r in res]
            res = None
        print(f"panel={on} C2 sequence ms {ts} ortho {ortho:.1f} ms loops {loops}", flush=True)
lib.chfsi_set_panel_kernels(1)
