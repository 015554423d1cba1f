"""Find the first phase whose output differs between identical solves."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1206_3768_b200 as pkg
import paper_1206_3768_b200.chfsi as ch
from paper_1206_3768_b200.harness import default_config
cfg_b = pkg.BASELINE_CONFIGS["C2"]
cfg = default_config(cfg_b)
seq = list(pkg.iter_baseline_sequence(cfg_b.n, 3, seed=0))
res = pkg.solve_sequence(seq[:2], cfg, mode="chained")
r = res[-1]
guess = pkg.ChfsiGuess(vectors=r.report.tail_vectors.clone(), lambda1=float(r.values[0]),
                       lambda_blk_plus_1=float(r.report.lambda_blk_plus_1))
sp = pkg.to_standard(pkg.EigenPencil(a=seq[2][1], b=seq[2][2], label=3))
trace = []
of, oo, orr = ch._filter_into, ch._orthonormalize_panel, ch._rr_core
def f(*a, **k):
    out = of(*a, **k); trace.append(("filter", out.clone())); return out
def o(work, *a, **k):
    trace.append(("pre_qr", work.clone())); out = oo(work, *a, **k); trace.append(("qr", work.clone())); return out
def rr(op, panel, hp, g, rot_p, rot_hp, ritz_d, res_d):
    orr(op, panel, hp, g, rot_p, rot_hp, ritz_d, res_d)
    trace.append(("hp", hp.clone())); trace.append(("gram_eig", g.clone())); trace.append(("ritz", ritz_d.clone())); trace.append(("rot", rot_p.clone()))
ch._filter_into, ch._orthonormalize_panel, ch._rr_core = f, o, rr
runs = []
for it in range(4):
    trace.clear()
    sol, rep = pkg.chfsi_solve(sp.h, cfg, guess=guess, rng=np.random.default_rng((0, 3, 1)))
    runs.append(list(trace)); print("run", it, rep.inner_loops, flush=True)
for it in range(1, 4):
    for idx, ((n0, t0), (n1, t1)) in enumerate(zip(runs[0], runs[it])):
        if t0.shape != t1.shape or not torch.equal(t0, t1):
            print("run", it, "first difference at step", idx, n0, "max abs diff", float((t0 - t1).abs().max()) if t0.shape == t1.shape else "shape")
            break
    else:
        print("run", it, "identical")
