"""GPU busy/idle breakdown of one chained sequence (CUPTI via torch.profiler).

    python tools/diag/gpu_idle.py [--config C2] [--top 25]

Prints the wall span, the union of kernel/memcpy intervals, and the idle
gaps grouped by (previous kernel -> next kernel), largest total first: the
host-overhead / sync bubbles of the solver loop.
"""
import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch
from torch.profiler import ProfilerActivity, profile

import paper_1206_3768_b200 as pkg
from paper_1206_3768_b200.harness import default_config, solve_sequence

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--problems", type=int, default=None)
a = ap.parse_args()

cfg_b = pkg.BASELINE_CONFIGS[a.config]
cfg = default_config(cfg_b)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, a.problems or cfg_b.length, seed=0))
dev = torch.device("cuda", 0)
pencils = [pkg.EigenPencil(a=torch.from_numpy(x).to(dev), b=torch.from_numpy(y).to(dev), label=lab)
           for lab, x, y in seq]
for _ in range(2):
    solve_sequence(pencils, cfg, seed=0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    solve_sequence(pencils, cfg, seed=0)
    torch.cuda.synchronize()

evs = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start:
        evs.append((e.time_range.start, e.time_range.end, e.name))
evs.sort()
if not evs:
    sys.exit("no device events captured")
span = evs[-1][1] - evs[0][0]
busy = 0.0
cur_s, cur_e = evs[0][0], evs[0][1]
gaps = collections.defaultdict(lambda: [0, 0.0])
prev_name = evs[0][2]
per_kernel = collections.defaultdict(lambda: [0, 0.0])
for s, e, name in evs:
    per_kernel[name][0] += 1
    per_kernel[name][1] += e - s
for s, e, name in evs[1:]:
    if s > cur_e:
        busy += cur_e - cur_s
        g = s - cur_e
        key = (prev_name[:60], name[:60])
        gaps[key][0] += 1
        gaps[key][1] += g
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
    prev_name = name
busy += cur_e - cur_s
print(f"span {span / 1e3:.2f} ms  busy {busy / 1e3:.2f} ms  idle {(span - busy) / 1e3:.2f} ms "
      f"({100 * (span - busy) / span:.1f}%)  events {len(evs)}")
print("\nidle gaps by (prev -> next), total ms, count:")
for (p, n), (c, t) in sorted(gaps.items(), key=lambda kv: -kv[1][1])[: a.top]:
    print(f"{t / 1e3:9.3f} {c:6d}  {p}  ->  {n}")
print("\nkernels by total device time (ms, count):")
for name, (c, t) in sorted(per_kernel.items(), key=lambda kv: -kv[1][1])[: a.top]:
    print(f"{t / 1e3:9.3f} {c:6d}  {name[:110]}")

# host activity during device-idle gaps: CPU ops / runtime calls overlapping
# each gap of >= 20 us, overlap time summed per name (nested ops both count)
cpu = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
             if e.device_type == torch.autograd.DeviceType.CPU)
idle = []
cur_e = evs[0][1]
for s, e, name in evs[1:]:
    if s > cur_e + 20:
        idle.append((cur_e, s))
    cur_e = max(cur_e, e)
host = collections.defaultdict(lambda: [0, 0.0])
import bisect
starts = [c[0] for c in cpu]
maxlen = max((c[1] - c[0] for c in cpu), default=0)
for gs, ge in idle:
    i = bisect.bisect_left(starts, gs - maxlen)
    seen = set()
    while i < len(cpu) and cpu[i][0] < ge:
        cs, ce, name = cpu[i]
        ov = min(ce, ge) - max(cs, gs)
        if ov > 0:
            host[name][1] += ov
            if name not in seen:
                host[name][0] += 1
                seen.add(name)
        i += 1
print(f"\nhost ops overlapping device-idle gaps >= 20 us ({len(idle)} gaps, "
      f"{sum(g - s for s, g in idle) / 1e3:.2f} ms):")
for name, (c, t) in sorted(host.items(), key=lambda kv: -kv[1][1])[: a.top]:
    print(f"{t / 1e3:9.3f} {c:6d}  {name[:110]}")
