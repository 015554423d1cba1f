"""In-situ kernel time of one chained sequence, by kernel and by stream
(CUPTI via torch.profiler; not serialised like an ncu launch list).

    python tools/diag/kernel_mix.py [--config C2] [--top 40] [--json out.json]

Prints per kernel name: launches, total and mean device time, stream ids;
then per stream the busy time, and the main stream's span / busy / idle.
"""
import argparse
import collections
import json
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
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--problems", type=int, default=None)
ap.add_argument("--json", default=None)
ap.add_argument("--by-stream", action="store_true", help="one row per (kernel, stream)")
a = ap.parse_args()

cfg_b = pkg.BASELINE_CONFIGS[a.config]
cfg = default_config(cfg_b)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, a.problems or cfg_b.length, seed=0, device=0))
pencils = [pkg.EigenPencil(a=x, b=y, label=lab) for lab, x, y in seq]
for _ in range(3):
    solve_sequence(pencils, cfg, seed=0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    res = solve_sequence(pencils, cfg, seed=0)
    torch.cuda.synchronize()

kern = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
by = collections.defaultdict(lambda: [0, 0.0, set()])
streams = collections.defaultdict(list)
for e in kern:
    name = e.name
    st = getattr(e, "device_resource_id", None)
    ivl = (e.time_range.start, e.time_range.end)
    rec = by[(name[:100] + f"  @s{st}") if a.by_stream else name[:110]]
    rec[0] += 1
    rec[1] += ivl[1] - ivl[0]
    rec[2].add(st)
    streams[st].append(ivl)
tot = sum(v[1] for v in by.values())
print(f"{len(kern)} device activities, {tot / 1e3:.2f} ms summed")
rows = sorted(by.items(), key=lambda kv: -kv[1][1])
for name, (cnt, us, sts) in rows[: a.top]:
    print(f"{us / 1e3:9.3f} ms {100 * us / tot:5.1f}% {cnt:6d}x {us / cnt:8.1f} us  s{sorted(sts)}  {name}")


def union(ivls):
    ivls = sorted(ivls)
    busy, cur_s, cur_e = 0.0, None, None
    for s, e in ivls:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        busy += cur_e - cur_s
    return busy, ivls[0][0], max(e for _, e in ivls)


for st, ivls in sorted(streams.items(), key=lambda kv: -len(kv[1])):
    busy, s0, s1 = union(ivls)
    print(f"stream {st}: {len(ivls)} activities, busy {busy / 1e3:.2f} ms of span {(s1 - s0) / 1e3:.2f} ms")
allb, s0, s1 = union([i for v in streams.values() for i in v])
print(f"all streams: busy {allb / 1e3:.2f} ms of span {(s1 - s0) / 1e3:.2f} ms "
      f"(idle {(s1 - s0 - allb) / 1e3:.2f} ms)")
phase = collections.Counter()
for r in res:
    for k in ("t_lanczos", "t_filter", "t_ortho", "t_rr"):
        phase[k] += getattr(r.report, k) * 1e3
print("solver phases (ms): " + ", ".join(f"{k} {v:.1f}" for k, v in phase.items()))
if a.json:
    json.dump({"kernels": [[n, c, u] for n, (c, u, _) in rows], "phases": dict(phase)},
              open(a.json, "w"), indent=1)

# main-stream idle gaps attributed to (previous -> next) activity
main_st = max(streams, key=lambda s: len(streams[s]))
mk = sorted((e.time_range.start, e.time_range.end, e.name) for e in kern
            if getattr(e, "device_resource_id", None) == main_st)
gaps = collections.defaultdict(lambda: [0, 0.0])
cur_e, prev = mk[0][1], mk[0][2]
hist = collections.Counter()
for s_, e_, name in mk[1:]:
    g = s_ - cur_e
    if g > 0:
        key = (prev[:55], name[:55])
        gaps[key][0] += 1
        gaps[key][1] += g
        hist[min(int(g // 10) * 10, 200)] += 1
    cur_e = max(cur_e, e_)
    prev = name
tot_gap = sum(v[1] for v in gaps.values())
print(f"\nmain stream {main_st}: {tot_gap / 1e3:.2f} ms idle in {sum(v[0] for v in gaps.values())} gaps; "
      f"gap histogram (us bucket: count) {sorted(hist.items())}")
for (p, n), (c, t) in sorted(gaps.items(), key=lambda kv: -kv[1][1])[: a.top]:
    print(f"{t / 1e3:8.3f} ms {c:6d}x {t / c:7.1f} us  {p}  ->  {n}")
