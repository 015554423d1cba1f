"""Live n x n device tensors after repeated C1 sequence calls, and who
holds them (leak hunt for the sequence driver)."""
import gc
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch

import paper_1206_3768_b200 as pkg

cfg_b = pkg.BASELINE_CONFIGS["C1"]
cfg = pkg.ChfsiConfig(nev=cfg_b.nev, nex=cfg_b.nex, deg=cfg_b.deg, tol=cfg_b.tol)
dev = torch.device("cuda", 0)
n = cfg_b.n
seq = [pkg.EigenPencil(a=torch.from_numpy(a).to(dev), b=torch.from_numpy(b).to(dev), label=lab)
       for lab, a, b in pkg.iter_baseline_sequence(n, 6, seed=0)]


def big():
    return [o for o in gc.get_objects()
            if isinstance(o, torch.Tensor) and o.is_cuda and o.numel() >= n * n]


for call in range(4):
    pkg.solve_sequence(seq, cfg, seed=0)
    gc.collect()
    torch.cuda.synchronize()
    ts = big()
    print(call, torch.cuda.memory_allocated(dev) >> 10, "KB, big tensors:", len(ts), flush=True)
ts = big()
inputs = {id(p.a) for p in seq} | {id(p.b) for p in seq}
for t in ts:
    if id(t) in inputs:
        continue
    refs = [type(r).__name__ + (":" + ",".join(str(k) for k in list(r.keys())[:6]) if isinstance(r, dict) else "")
            for r in gc.get_referrers(t) if r is not ts]
    print("tensor", tuple(t.shape), t.untyped_storage().nbytes() >> 10, "KB held by", refs[:5])
