"""Goldens for the `run_experiment` drop-in and the reference generator.

Runs the UNMODIFIED reference (`spectral_chain`, imported read-only from
/root/reference/pkg/src; only in the build container) on small specs and
writes `experiment.npz`:

* per spec: the ExperimentReport rows (counts, medians, residual maxima,
  convergence flags), `blk` and the warnings; once, the CSV column schema
  `REPORT_FIELDS` that `emit_report` writes (harness.py:52-65);
* the reference generator's bytes: SHA-256 and an entry probe of every A/B
  of each spec's sequence (`generate_sequence`, sequence.py:137-178), so the
  CPU suite proves `sequence.iter_generated_sequence` draws the same
  matrices;
* `match_eigenvectors` on the dense solutions of adjacent problems
  (sequence.py:187-220): sigma and theta, pinning the device matcher.

    python tests/golden/make_golden_experiment.py     # ~10 s
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import spectral_chain as sc  # noqa: E402  (the reference, read-only)
from spectral_chain import harness as sch  # noqa: E402

from tests.golden.recipes import sha  # noqa: E402

# (name, n, schedule kwargs, seed, nev, overrides, tracked_fraction)
SPECS = [
    ("gen96", 96, dict(length=4), 3, 8, dict(deg=10), 1.0),
    ("gen130", 130, dict(length=3, eps=[0.05, 0.01]), 5, 6, dict(blk=20, deg=14, tol=1e-9), 0.5),
    ("gen64_nob", 64, dict(length=3, perturb_b=False, b_cond_target=50.0), 11, 5, dict(blk=16), 1.0),
]
ROW_INT = ["matvecs_random", "matvecs_approx", "filtered_random", "filtered_approx",
           "inner_loops_random", "inner_loops_approx", "ell"]
ROW_FLOAT = ["median_angle", "max_residual_random", "max_residual_approx", "speedup_matvec"]
ROW_BOOL = ["converged_random", "converged_approx"]


def main():
    out = {"names": np.asarray([s[0] for s in SPECS]),
           "report_fields": np.asarray(sch.REPORT_FIELDS)}
    for name, n, sched, seed, nev, over, frac in SPECS:
        schedule = sc.CorrelationSchedule(**sched)
        spec = sch.ExperimentSpec(source=sch.GenerateSource(n=n, schedule=schedule, seed=seed),
                                  solver="chfsi", nev=nev, solver_overrides=over,
                                  tracked_fraction=frac, repetitions=1, seed=seed)
        rep = sch.run_experiment(spec)
        pre = f"{name}/"
        out[pre + "spec"] = np.bytes_(json.dumps(dict(n=n, schedule=sched, seed=seed, nev=nev,
                                                      overrides=over, fraction=frac)))
        out[pre + "blk"] = np.int64(rep.blk)
        out[pre + "warnings"] = np.bytes_(json.dumps(rep.warnings))
        for k in ROW_INT:
            out[pre + k] = np.asarray([getattr(r, k) for r in rep.rows], dtype=np.int64)
        for k in ROW_FLOAT:
            out[pre + k] = np.asarray([getattr(r, k) for r in rep.rows], dtype=np.float64)
        for k in ROW_BOOL:
            out[pre + k] = np.asarray([getattr(r, k) for r in rep.rows], dtype=bool)
        seq = sc.generate_sequence(n, schedule, seed=seed)
        for p in seq.pencils:
            out[pre + f"a_sha/{p.label}"] = np.bytes_(sha(p.a))
            out[pre + f"b_sha/{p.label}"] = np.bytes_(sha(p.b))
            out[pre + f"a_probe/{p.label}"] = p.a[::7, ::5].copy()
            out[pre + f"b_probe/{p.label}"] = p.b[::7, ::5].copy()
        # match_eigenvectors on adjacent dense solutions (tracked columns)
        blk = rep.blk
        keep = max(blk + 1, nev)
        tracked = max(1, int(np.ceil(frac * nev)))
        sols = [sch.oracle_solve(p, keep)[0] for p in seq.pencils]
        for i in range(len(sols) - 1):
            sigma, theta = sc.match_eigenvectors(sch.replace_tracked(sols[i], tracked), None,
                                                 sch.replace_tracked(sols[i + 1], tracked), None)
            out[pre + f"sigma/{i + 1}"] = sigma.astype(np.int64)
            out[pre + f"theta/{i + 1}"] = theta
        print(f"{name}: blk {rep.blk}, rows " + ", ".join(
            f"l{r.ell}: mv {r.matvecs_random}/{r.matvecs_approx} loops "
            f"{r.inner_loops_random}/{r.inner_loops_approx}" for r in rep.rows), flush=True)
    path = os.path.join(HERE, "experiment.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.1f} kB)")


if __name__ == "__main__":
    main()
