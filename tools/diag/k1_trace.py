"""Per-CTA timeline of one K1 launch (CHFSI_K1_DEBUG=8).

    CHFSI_K1_DEBUG=8 python tools/diag/k1_trace.py --n 4096 --w 160
Prints the CTA end-time distribution, the owner waits, and the slowest CTAs.
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200 import _lib
from paper_1206_3768_b200._device import Operator, fblock
from paper_1206_3768_b200.chfsi import _filter_into

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--w", type=int, default=160)
ap.add_argument("--bn", type=int, default=0)
ap.add_argument("--groups", type=int, default=1)
a = ap.parse_args()
assert int(os.environ.get("CHFSI_K1_DEBUG", "0")) & 8, "run with CHFSI_K1_DEBUG=8"
g = torch.randn(a.n, a.n, dtype=torch.complex128, device="cuda")
op = Operator((g + g.conj().T) / 2)
y = fblock(a.n, a.w)
y.copy_(torch.randn(a.n, a.w, dtype=torch.complex128, device="cuda"))
x = fblock(a.n, a.w)
if a.bn:
    _lib.check(_lib.lib().chfsi_ctx_set_tiling(_lib.ctx(), 64, a.bn, 0))
    if a.groups != 1:
        _lib.check(_lib.lib().chfsi_ctx_set_step_groups(_lib.ctx(), a.groups))
win = pkg.FilterWindow(a=-5.0, b=60.0, scale_ref=-70.0)
for _ in range(3):
    _filter_into(op, y, x, y, 1, win)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (5 * 4096))()
n = _lib.lib().chfsi_debug_k1_trace(buf, 4096)
t = np.array(buf[: 5 * n], dtype=np.float64).reshape(n, 5)
t0 = t[:, 0].min()
start, wb, we, end = (t[:, 0] - t0) / 1e3, t[:, 1], t[:, 2], (t[:, 3] - t0) / 1e3
raw = t[:, 4].astype(np.int64)
sm, bidx = raw & 0xFFFF, raw >> 16
wait = np.where(wb > 0, (we - wb) / 1e3, 0.0)
print(f"ctas {n}  start max {start.max():.1f} us  end min/med/max {end.min():.1f}/"
      f"{np.median(end):.1f}/{end.max():.1f} us  owner wait max {wait.max():.1f} us")
order = np.argsort(-end)
for c in order[:12]:
    print(f"cta {c:4d} sm {int(sm[c]):3d} start {start[c]:7.1f} end {end[c]:7.1f} wait {wait[c]:7.1f}")
hist = np.histogram(end, bins=10)
print("end histogram:", list(hist[0]), [round(v, 1) for v in hist[1]])
# co-residency: which CTAs share an SM, and which of the pair finishes first
pairs = {}
for c in range(n):
    pairs.setdefault(int(sm[c]), []).append(c)
lower_first = same_offset = npairs = 0
for s_, cs in pairs.items():
    if len(cs) != 2:
        continue
    npairs += 1
    lo, hi = sorted(cs, key=lambda c: bidx[c])  # by hardware blockIdx
    lower_first += end[lo] < end[hi]
    same_offset += abs(int(bidx[hi]) - int(bidx[lo])) == n // 2
print(f"SMs with 2 CTAs: {npairs}/{len(pairs)}; lower blockIdx ends first: {lower_first}; "
      f"pair is (c, c+grid/2): {same_offset}")
early = end < np.median(end)
print("early CTAs with blockIdx < grid/2:", int(np.sum(early & (bidx < n // 2))), "of", int(early.sum()))
print("early CTAs with logical index < grid/2:", int(np.sum(early[: n // 2])), "of", int(early.sum()))
