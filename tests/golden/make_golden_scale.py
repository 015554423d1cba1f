"""Reference goldens at BASELINE scale (C2 chained, C3 x12, C4 x2, C5 x1).

Runs the UNMODIFIED reference `spectral_chain` (imported read-only from
/root/reference/pkg/src; this script only runs in the build container, the
GPU box never reads /root/reference) on the BASELINE generator
(`paper_1206_3768_b200.sequence`, host path) and writes small .npz
fixtures: eigenvalues, residuals, the reference's work counters, the dense
oracle's eigenvalues, input fingerprints and, per iterative cell, the
principal-angle sine between the reference ChFSI eigenspace and the dense
oracle eigenspace. Eigenvectors at these sizes are 40 MB - 1 GB per problem
and are NOT stored; the GPU tests bound the angle to the reference
eigenspace through the dense eigenspace instead (triangle inequality:
sin(gpu, ref) <= sin(gpu, dense_gpu) + d(dense_gpu, dense_cpu) +
sin(dense_cpu, ref), the middle term bounded by both dense solves'
residuals over the gap, see tests/test_gpu_scale.py).

Cells follow the reference harness (`harness.py:188-289`): for problem l
the dense oracle (`oracle_solve`, harness.py:149-161), a random-start ChFSI
with rng (0, l, 0) and, for l >= 2, a warm start from the dense oracle of
problem l-1 with rng (0, l, 1) (harness.py:235-255). `--c3` additionally
runs the oracle's chained driver (the restatement in
`oracle/chfsi_oracle.py`, pinned to the reference by test_oracle_golden)
warm-starting every problem from the previous ChFSI tail block.

Each file is rewritten after every finished cell, so a long run leaves
usable partial fixtures; `done_cells` lists what is in it.

    python tests/golden/make_golden_scale.py --c2-chained   # ~1 min
    python tests/golden/make_golden_scale.py --c3           # ~45 min on 8 cores
    python tests/golden/make_golden_scale.py --c4           # ~1-1.5 h
    python tests/golden/make_golden_scale.py --c5           # ~3-4 h, ~45 GB RAM
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import scipy.linalg

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import spectral_chain as sc  # noqa: E402  (the reference, read-only)

from oracle import chfsi_oracle as orc  # noqa: E402
from tests.golden.recipes import sha  # noqa: E402
from paper_1206_3768_b200.sequence import BASELINE_CONFIGS, iter_baseline_sequence  # noqa: E402

PROBE = (97, 89)  # entry fingerprint stride (the GPU box regenerates the inputs)


def sines(u, v):
    """Principal-angle sines (reference test helper, test_chfsi.py:31-33)."""
    return np.linalg.svd(v - u @ (u.conj().T @ v), compute_uv=False)


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


class Fixture:
    """An .npz rewritten after every cell."""

    def __init__(self, name, **meta):
        self.path = os.path.join(HERE, name)
        self.data = dict(meta)
        self.done = []
        self.timings = {}

    def cell(self, key, seconds, **arrays):
        self.data.update(arrays)
        self.done.append(key)
        self.timings[key] = round(seconds, 2)
        self.data["done_cells"] = np.asarray(self.done)
        self.data["timings_json"] = np.bytes_(json.dumps(self.timings))
        tmp = self.path + ".tmp.npz"
        np.savez_compressed(tmp, **self.data)
        os.replace(tmp, self.path)
        print(f"[{time.strftime('%H:%M:%S')}] {os.path.basename(self.path)} {key}: "
              f"{seconds:.1f} s ({os.path.getsize(self.path) / 1e3:.0f} kB)", flush=True)


def input_cell(fx, label, a, b):
    fx.cell(f"{label}/input", 0.0, **{
        f"{label}/a_sha": np.bytes_(sha(a)),
        f"{label}/b_sha": np.bytes_(sha(b)),
        f"{label}/a_probe": a[:: PROBE[0], :: PROBE[1]].copy(),
        f"{label}/b_probe": b[:: PROBE[0], :: PROBE[1]].copy(),
    })


def dense_cell(fx, label, h, nev, blk, subset=False):
    """Dense oracle of the standard problem (harness.oracle_solve's eigh).

    ``subset``: only the lowest blk+1 pairs via LAPACK zheevr (C5, where
    the full n x n eigenvector matrix would not fit next to H in host RAM);
    the same eigenpairs to rounding as the full zheevd.
    """
    t0 = time.perf_counter()
    if subset:
        vals, vecs = scipy.linalg.eigh(h, subset_by_index=[0, blk], driver="evr",
                                       check_finite=False)
    else:
        vals, vecs = sc.hermitian_eig(h)
    vecs = np.asfortranarray(vecs[:, : blk + 1]) if not subset else vecs
    dense_res = np.linalg.norm(h @ vecs[:, :nev] - vecs[:, :nev] * vals[:nev], axis=0)
    fx.cell(f"{label}/dense", time.perf_counter() - t0, **{
        f"{label}/dense_values": np.asarray(vals[: blk + 1]),
        f"{label}/dense_residuals": dense_res,
        f"{label}/dense_h_norm_est": np.float64(max(abs(vals[0]), abs(vals[-1]))),
    })
    return vals[: blk + 1], vecs[:, : blk + 1]


def solve_cell(fx, label, kind, h, ccfg, guess, seed, dense_vecs, nev):
    t0 = time.perf_counter()
    sol, rep = sc.chfsi_solve(h, ccfg, guess=guess, rng=np.random.default_rng(seed), label=label)
    dt = time.perf_counter() - t0
    pre = f"{label}/{kind}/"
    arrays = report_arrays(pre, rep)
    arrays[pre + "values"] = sol.values
    arrays[pre + "dense_sine"] = np.float64(sines(dense_vecs[:, :nev], sol.vectors).max())
    fx.cell(f"{label}/{kind}", dt, **arrays)
    return sol, rep


def chained_cell(fx, label, h, cfg, prev, dense_vecs):
    """The oracle's chained driver step (orc.run_sequence(mode="chained"))."""
    t0 = time.perf_counter()
    rng = np.random.default_rng((0, label, 0) if prev is None else (0, label, 1))
    vals, vecs, rep = orc.chfsi_solve(h, cfg.nev, cfg.blk, cfg.deg, cfg.tol, guess=prev, rng=rng)
    dt = time.perf_counter() - t0
    pre = f"{label}/chained/"
    arrays = {
        pre + "values": vals,
        pre + "inner_loops": np.int64(rep.inner_loops),
        pre + "filtered_vectors": np.int64(rep.filtered_vectors),
        pre + "matvecs": np.int64(rep.matvecs),
        pre + "lanczos_matvecs": np.int64(rep.lanczos_matvecs),
        pre + "locked_per_loop": np.asarray(rep.locked_per_loop, dtype=np.int64),
        pre + "final_residuals": np.asarray(rep.final_residuals),
        pre + "converged": np.bool_(rep.converged),
        pre + "lambda_blk_plus_1": np.float64(rep.lambda_blk_plus_1),
        pre + "dense_sine": np.float64(sines(dense_vecs[:, : cfg.nev], vecs).max()),
    }
    fx.cell(f"{label}/chained", dt, **arrays)
    return (rep.tail_vectors, float(vals[0]), rep.lambda_blk_plus_1), vals


def harness_sequence(cfg_name, limit, chained, cold_labels=None, order=None):
    cfg = BASELINE_CONFIGS[cfg_name]
    ccfg = sc.ChfsiConfig(nev=cfg.nev, blk=cfg.blk, deg=cfg.deg, tol=cfg.tol)
    fx = Fixture(f"{cfg_name.lower()}_scale.npz", n=np.int64(cfg.n), length=np.int64(cfg.length),
                 nev=np.int64(cfg.nev), blk=np.int64(cfg.blk), deg=np.int64(cfg.deg),
                 probe_stride=np.asarray(PROBE, dtype=np.int64),
                 protocol=np.bytes_("harness.py:188-289 cells + oracle chained" if chained
                                    else "harness.py:188-289 cells"))
    prev_dense = None
    prev_chain = None
    for label, a, b in iter_baseline_sequence(cfg.n, cfg.length, seed=0):
        if label > limit:
            break
        input_cell(fx, label, a, b)
        t0 = time.perf_counter()
        sp = sc.to_standard(sc.EigenPencil(a=a, b=b, label=label))
        del a, b
        fx.cell(f"{label}/reduce", time.perf_counter() - t0,
                **{f"{label}/h_probe": sp.h[:: PROBE[0], :: PROBE[1]].copy()})
        h = sp.h
        dvals, dvecs = dense_cell(fx, label, h, cfg.nev, cfg.blk)
        cells = order or ["warm", "cold", "chained"]
        for kind in cells:
            if kind == "warm" and prev_dense is not None:
                pv, pvec = prev_dense
                guess = sc.ChfsiGuess(vectors=pvec[:, : cfg.blk], lambda1=float(pv[0]),
                                      lambda_blk_plus_1=float(pv[cfg.blk]))
                solve_cell(fx, label, "warm", h, ccfg, guess, (0, label, 1), dvecs, cfg.nev)
            elif kind == "cold" and (cold_labels is None or label in cold_labels):
                solve_cell(fx, label, "cold", h, ccfg, None, (0, label, 0), dvecs, cfg.nev)
            elif kind == "chained" and chained:
                prev_chain, _ = chained_cell(fx, label, h, cfg, prev_chain, dvecs)
        prev_dense = (dvals, dvecs)
        del sp, h


def c5_problem1():
    """C5 problem 1 (cold) at FIXED degree 36 (adaptive degree
    has no reference; eigenpair parity is pinned at the cap instead)."""
    cfg = BASELINE_CONFIGS["C5"]
    ccfg = sc.ChfsiConfig(nev=cfg.nev, blk=cfg.blk, deg=cfg.deg, tol=cfg.tol)
    fx = Fixture("c5_scale.npz", n=np.int64(cfg.n), length=np.int64(1), nev=np.int64(cfg.nev),
                 blk=np.int64(cfg.blk), deg=np.int64(cfg.deg),
                 probe_stride=np.asarray(PROBE, dtype=np.int64),
                 protocol=np.bytes_("problem 1 random-start cell, fixed deg 36; dense via zheevr"))
    t0 = time.perf_counter()
    gen = iter_baseline_sequence(cfg.n, 1, seed=0)
    label, a, b = next(gen)
    gen.close()
    fx.cell("1/generate", time.perf_counter() - t0)
    input_cell(fx, 1, a, b)
    t0 = time.perf_counter()
    pencil = sc.EigenPencil(a=a, b=b, label=1)
    del a, b
    sp = sc.to_standard(pencil)
    del pencil
    h = sp.h
    l_probe = sp.cholesky_factor[:: PROBE[0], :: PROBE[1]].copy()
    del sp
    fx.cell("1/reduce", time.perf_counter() - t0,
            **{"1/h_probe": h[:: PROBE[0], :: PROBE[1]].copy(), "1/l_probe": l_probe})
    dvals, dvecs = dense_cell(fx, 1, h, cfg.nev, cfg.blk, subset=True)
    solve_cell(fx, 1, "cold", h, ccfg, None, (0, 1, 0), dvecs, cfg.nev)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--c2-chained", action="store_true")
    p.add_argument("--c3", action="store_true")
    p.add_argument("--c4", action="store_true")
    p.add_argument("--c5", action="store_true")
    args = p.parse_args()
    if args.c2_chained:
        harness_sequence("C2", 10, chained=True, cold_labels={1}, order=["chained"])
    if args.c3:
        harness_sequence("C3", 12, chained=True)
    if args.c4:
        harness_sequence("C4", 2, chained=False, order=["warm", "cold"])
    if args.c5:
        c5_problem1()


if __name__ == "__main__":
    main()
