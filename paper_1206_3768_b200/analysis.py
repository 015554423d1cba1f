"""Warm-start diagnostics on the device.

`match_eigenvectors` / `angle_report` restate the reference's eigenvector
correspondence (`sequence.py:187-257`): the cross-Gram
``|Y_prev^H Y_next|`` of standard-form vectors (``L^H x`` for generalized
solutions) is one ZGEMM on the device; the greedy one-to-one matching —
repeatedly take the largest remaining entry, never reusing a row or column
— is done on the host over the entries sorted once in descending order
(ties in row-major order, as ``np.argmax`` resolves them), O(m^2 log m)
instead of the reference's O(m^3) repeated argmax, same result.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from ._device import fblock, ld_of, to_fblock
from ._lib import check, ctx, dptr, lib
from .linalg import cholesky
from .reduction import forward_transform

__all__ = ["AngleReport", "match_eigenvectors", "angle_report"]


@dataclass
class AngleReport:
    """Per adjacent pair (keyed by the first label): angles, matching and the
    median angle (sequence.py:81-93 fields)."""

    angles: dict = field(default_factory=dict)
    matching: dict = field(default_factory=dict)
    median_angles: dict = field(default_factory=dict)


def _standard_vectors(sol, l_factor):
    if sol.form == "standard":
        return to_fblock(sol.vectors)
    return to_fblock(forward_transform(to_fblock(l_factor), to_fblock(sol.vectors)))


def greedy_match(gram):
    """sigma[i] = column matched to row i, largest-first, one-to-one."""
    m = gram.shape[0]
    flat = np.asarray(gram).ravel()
    order = np.argsort(-flat, kind="stable")  # descending, ties in row-major order
    sigma = np.full(m, -1, dtype=int)
    used_r = np.zeros(m, dtype=bool)
    used_c = np.zeros(m, dtype=bool)
    found = 0
    for idx in order:
        i, j = divmod(int(idx), m)
        if used_r[i] or used_c[j]:
            continue
        sigma[i] = j
        used_r[i] = used_c[j] = True
        found += 1
        if found == m:
            break
    return sigma


def match_eigenvectors(sol_prev, l_prev, sol_next, l_next):
    """One-to-one correspondence between adjacent solutions and the
    deviation angles arccos(min(1, |M[i, sigma[i]]|)) (sequence.py:187-220)."""
    y_prev = _standard_vectors(sol_prev, l_prev)
    y_next = _standard_vectors(sol_next, l_next)
    if y_prev.shape[0] != y_next.shape[0]:
        raise ValueError("solutions live in different dimensions")
    m = min(y_prev.shape[1], y_next.shape[1])
    n = y_prev.shape[0]
    g = fblock(m, m)
    check(lib().chfsi_gemm_z(ctx(), b"C", b"N", m, m, n, 1.0, 0.0, dptr(y_prev), ld_of(y_prev),
                             dptr(y_next), ld_of(y_next), 0.0, 0.0, dptr(g), ld_of(g)),
          "cross-Gram")
    gram = g.abs().cpu().numpy()
    sigma = greedy_match(gram)
    theta = np.arccos(np.minimum(1.0, gram[np.arange(m), sigma]))
    return sigma, theta


def angle_report(pencils, solutions, fraction=1.0):
    """Per-pair deviation angles along a sequence (sequence.py:223-257).
    ``pencils`` are EigenPencils (for the Cholesky factors of generalized
    solutions) in the same order as ``solutions``."""
    if not 0 < fraction <= 1:
        raise ValueError("fraction must be in (0, 1]")
    pencils = list(getattr(pencils, "pencils", pencils))  # a PencilSequence or pencils
    if len(solutions) != len(pencils):
        raise ValueError(f"need one solution per pencil ({len(pencils)}), got {len(solutions)}")
    report = AngleReport()
    factors = {}

    def factor(idx):
        if idx not in factors:
            factors[idx] = cholesky(pencils[idx].b)
        return factors[idx]

    for idx in range(len(pencils) - 1):
        sa, sb = solutions[idx], solutions[idx + 1]
        if sa is None or sb is None:
            raise ValueError(f"missing solution for adjacent labels {idx + 1}, {idx + 2}")
        tracked = max(1, int(math.ceil(fraction * min(sa.nev, sb.nev))))
        la = factor(idx) if sa.form == "generalized" else None
        lb = factor(idx + 1) if sb.form == "generalized" else None
        ta = replace(sa, values=sa.values[:tracked], vectors=sa.vectors[:, :tracked])
        tb = replace(sb, values=sb.values[:tracked], vectors=sb.vectors[:, :tracked])
        sigma, theta = match_eigenvectors(ta, la, tb, lb)
        report.angles[idx + 1] = theta
        report.matching[idx + 1] = sigma
        report.median_angles[idx + 1] = float(np.median(theta))
    return report
