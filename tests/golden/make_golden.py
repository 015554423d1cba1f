"""Generate the golden vectors that pin the oracle and the device path.

Runs the UNMODIFIED reference `spectral_chain` (imported read-only from
/root/reference/pkg/src — this script only runs in the build container; the
GPU box never reads /root/reference) on seeded inputs and writes compressed
.npz fixtures next to this file. Inputs that are cheap to regenerate are
stored as (seed, recipe) plus a SHA-256 of their bytes, so the tests can
rebuild them and prove they rebuilt the same bytes.

    python tests/golden/make_golden.py            # C1 + small cases
    python tests/golden/make_golden.py --c2       # also the n=2048 sequence
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import spectral_chain as sc  # noqa: E402  (the reference, read-only)

from tests.golden.recipes import (  # noqa: E402
    SOLVE_CASES,
    FILTER_CASES,
    LANCZOS_CASES,
    QR_CASES,
    REDUCTION_CASES,
    build_filter_case,
    build_lanczos_case,
    build_qr_case,
    build_reduction_case,
    build_solve_case,
    sha,
)
from paper_1206_3768_b200.sequence import BASELINE_CONFIGS, iter_baseline_sequence  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name} ({os.path.getsize(path) / 1e3:.1f} kB)")


def report_arrays(prefix, rep):
    return {
        f"{prefix}inner_loops": np.int64(rep.inner_loops),
        f"{prefix}filtered_vectors": np.int64(rep.filtered_vectors),
        f"{prefix}matvecs": np.int64(rep.matvecs),
        f"{prefix}lanczos_matvecs": np.int64(rep.lanczos_matvecs),
        f"{prefix}residual_check_matvecs": np.int64(rep.residual_check_matvecs),
        f"{prefix}locked_per_loop": np.asarray(rep.locked_per_loop, dtype=np.int64),
        f"{prefix}final_residuals": np.asarray(rep.final_residuals),
        f"{prefix}converged": np.bool_(rep.converged),
        f"{prefix}operator_norm_estimate": np.float64(rep.operator_norm_estimate),
    }


def small_cases():
    out = {}
    for name, spec in FILTER_CASES.items():
        h, y, (a, b, s), deg = build_filter_case(spec)
        ym = sc.chebyshev_filter(h, y, deg, sc.FilterWindow(a=a, b=b, scale_ref=s))
        out[f"filter/{name}/out"] = ym
        out[f"filter/{name}/h_sha"] = np.bytes_(sha(h))
        out[f"filter/{name}/y_sha"] = np.bytes_(sha(y))
        lam = np.linspace(s, b + 0.5, 41)
        out[f"filter/{name}/response"] = sc.chebyshev_response(
            lam, deg, sc.FilterWindow(a=a, b=b, scale_ref=s))
    for name, spec in LANCZOS_CASES.items():
        h, k, seed = build_lanczos_case(spec)
        ritz, beta_last, steps = sc.chfsi._lanczos_estimates(h, k, np.random.default_rng(seed))
        out[f"lanczos/{name}/ritz"] = ritz
        out[f"lanczos/{name}/beta_last"] = np.float64(beta_last)
        out[f"lanczos/{name}/steps"] = np.int64(steps)
        out[f"lanczos/{name}/bound"] = np.float64(
            sc.lanczos_upper_bound(h, k, rng=np.random.default_rng(seed)))
    for name, spec in QR_CASES.items():
        y = build_qr_case(spec)
        try:
            q = sc.qr_orthonormalize(y)
            out[f"qr/{name}/q"] = q
            out[f"qr/{name}/dead"] = np.zeros(0, dtype=np.int64)
        except sc.RankDeficientError as err:
            out[f"qr/{name}/dead"] = np.asarray(err.indices, dtype=np.int64)
    for name, spec in REDUCTION_CASES.items():
        a, b, y = build_reduction_case(spec)
        sp = sc.to_standard(sc.EigenPencil(a=a, b=b))
        sol = sc.back_transform(sp.cholesky_factor, sc.EigenSolution(values=np.zeros(y.shape[1]),
                                                                   vectors=y))
        out[f"reduction/{name}/h"] = sp.h
        out[f"reduction/{name}/l"] = sp.cholesky_factor
        out[f"reduction/{name}/x"] = sol.vectors
    for name, spec in SOLVE_CASES.items():
        h, cfg_kw, guess, seed = build_solve_case(spec)
        cfg = sc.ChfsiConfig(**cfg_kw)
        g = None if guess is None else sc.ChfsiGuess(vectors=guess[0], lambda1=guess[1],
                                                      lambda_blk_plus_1=guess[2])
        sol, rep = sc.chfsi_solve(h, cfg, guess=g, rng=np.random.default_rng(seed))
        out[f"solve/{name}/values"] = sol.values
        out[f"solve/{name}/vectors"] = sol.vectors
        for k, v in report_arrays(f"solve/{name}/", rep).items():
            out[k] = v
    save("small_cases.npz", **out)


def sequence_case(cfg_name, vector_labels, limit=None):
    """Reference harness protocol on the BASELINE generator (harness.py:188-289).

    For every problem: the dense oracle (to_standard + eigh), a cold ChFSI
    solve with rng (0, l, 0) and — for l >= 2 — a warm solve from the dense
    oracle of problem l-1 with rng (0, l, 1).
    """
    cfg = BASELINE_CONFIGS[cfg_name]
    ccfg = sc.ChfsiConfig(nev=cfg.nev, blk=cfg.blk, deg=cfg.deg, tol=cfg.tol)
    out = {"n": np.int64(cfg.n), "length": np.int64(cfg.length)}
    prev = None
    timings = {}
    for label, a, b in iter_baseline_sequence(cfg.n, cfg.length, seed=0):
        if limit is not None and label > limit:
            break
        out[f"{label}/a_sha"] = np.bytes_(sha(a))
        out[f"{label}/b_sha"] = np.bytes_(sha(b))
        # host-BLAS-independent fingerprint (the QR/GEMM of the generator
        # round differently on other CPUs; the GPU box checks these instead)
        out[f"{label}/a_probe"] = a[::37, ::41].copy()
        out[f"{label}/b_probe"] = b[::37, ::41].copy()
        t0 = time.perf_counter()
        pencil = sc.EigenPencil(a=a, b=b, label=label)
        sol_full, sp, vals = sc.oracle_solve(pencil, max(cfg.blk + 1, cfg.nev))
        out[f"{label}/dense_values"] = vals[: cfg.blk + 1]
        out[f"{label}/h_sha"] = np.bytes_(sha(sp.h))
        t1 = time.perf_counter()
        cold, rep_c = sc.chfsi_solve(sp.h, ccfg, rng=np.random.default_rng((0, label, 0)),
                                     label=label)
        t2 = time.perf_counter()
        out[f"{label}/cold/values"] = cold.values
        out.update(report_arrays(f"{label}/cold/", rep_c))
        if label in vector_labels:
            out[f"{label}/cold/vectors"] = cold.vectors
        timings[f"{label}/dense"] = t1 - t0
        timings[f"{label}/cold"] = t2 - t1
        if prev is not None:
            psol, pvals = prev
            guess = sc.ChfsiGuess(vectors=psol.vectors[:, : cfg.blk], lambda1=float(pvals[0]),
                                  lambda_blk_plus_1=float(pvals[cfg.blk]))
            t3 = time.perf_counter()
            warm, rep_w = sc.chfsi_solve(sp.h, ccfg, guess=guess,
                                         rng=np.random.default_rng((0, label, 1)), label=label)
            timings[f"{label}/warm"] = time.perf_counter() - t3
            out[f"{label}/warm/values"] = warm.values
            out.update(report_arrays(f"{label}/warm/", rep_w))
            if label in vector_labels:
                out[f"{label}/warm/vectors"] = warm.vectors
        prev = (sol_full, vals)
        print(f"{cfg_name} problem {label}: " + json.dumps(
            {k: round(v, 3) for k, v in timings.items() if k.startswith(f"{label}/")}))
    out["timings_json"] = np.bytes_(json.dumps(timings))
    save(f"{cfg_name.lower()}_harness.npz", **out)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--c2", action="store_true")
    p.add_argument("--skip-small", action="store_true")
    p.add_argument("--c3", action="store_true", help="C3 problems 1-3 (~10 min)")
    args = p.parse_args()
    if not args.skip_small:
        small_cases()
        sequence_case("C1", vector_labels={1, 2})
    if args.c2:
        sequence_case("C2", vector_labels=set())
    if args.c3:
        sequence_case("C3", vector_labels=set(), limit=3)


if __name__ == "__main__":
    main()
