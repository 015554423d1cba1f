"""First (problem, phase) whose output differs between identical chained C2 sequences."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1206_3768_b200 as pkg
import paper_1206_3768_b200.chfsi as ch
import paper_1206_3768_b200.harness as hs
from paper_1206_3768_b200.harness import default_config
cfg_b = pkg.BASELINE_CONFIGS["C2"]
cfg = default_config(cfg_b)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, cfg_b.length, seed=0))
dev = torch.device("cuda", 0)
pencils = [pkg.EigenPencil(a=torch.from_numpy(a).to(dev), b=torch.from_numpy(b).to(dev), label=l) for l, a, b in seq]
trace = []
def wrap(name, fn, out_arg=None):
    def w(*a, **k):
        out = fn(*a, **k)
        t = out if out_arg is None else a[out_arg]
        if isinstance(t, tuple): t = torch.tensor(np.asarray(t[0], dtype=float))
        if hasattr(t, "h"): t = t.h
        trace.append((name, t.clone()))
        return out
    return w
ch._filter_into = wrap("filter", ch._filter_into)
ch._orthonormalize_panel = wrap("qr", ch._orthonormalize_panel, 0)
ch._rr_core = wrap("rr_rot", ch._rr_core, 4)
ch._lanczos_estimates = wrap("lanczos", ch._lanczos_estimates)
hs.to_standard = wrap("to_standard_h", hs.to_standard)
runs = []
for it in range(5):
    trace.clear()
    res = pkg.solve_sequence(pencils, cfg, mode="chained")
    runs.append((list(trace), [r.report.inner_loops for r in res]))
    print("run", it, runs[-1][1], flush=True)
for it in range(1, 5):
    for idx, ((n0, t0), (n1, t1)) in enumerate(zip(runs[0][0], runs[it][0])):
        eq = t0.shape == t1.shape and torch.equal(t0, t1)
        if not eq:
            prob = sum(1 for n, _ in runs[0][0][:idx + 1] if n == "to_standard_h")
            names = [n for n, _ in runs[0][0][idx - 6: idx + 1]]
            d = float((t0 - t1).abs().max()) if t0.shape == t1.shape else -1
            print("run", it, "first difference at trace step", idx, n0, "problem", prob, "maxdiff", d, "context", names)
            break
    else:
        print("run", it, "identical")
