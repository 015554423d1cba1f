"""Deterministic input recipes shared by make_golden.py and the tests.

Every input is rebuilt from a numpy seed; the golden files store the
SHA-256 of the bytes so a test can prove it rebuilt exactly what the
reference saw. Case shapes mirror the reference's own tests
(`pkg/tests/test_chfsi.py`, `test_linalg.py`, `test_reduction.py`) plus
ragged sizes that are not multiples of any kernel tile.
"""

from __future__ import annotations

import hashlib

import numpy as np


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_hermitian(rng, n, scale=1.0):
    """Same recipe as the reference fixture `pkg/tests/conftest.py:5-7`."""
    g = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2)
    return scale * (g + g.conj().T) / 2


def random_spd(rng, n, cond=100.0):
    """Same recipe as `pkg/tests/conftest.py:10-16`."""
    g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    q, _ = np.linalg.qr(g)
    vals = np.logspace(0.0, np.log10(cond), n)
    m = (q * vals) @ q.conj().T
    return (m + m.conj().T) / 2


def cgauss(rng, n, m):
    return rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))


# ------------------------------------------------------------------ filter ---
FILTER_CASES = {
    # test_chfsi.py:69-78 — eigenbasis input, window (w[20], w[-1]+0.5, w[0])
    **{f"eig60_deg{d}": dict(kind="eig", n=60, seed=1234, deg=d) for d in (1, 8, 25, 40)},
    "rand96_w12_deg5": dict(kind="rand", n=96, w=12, seed=5, deg=5, ia=12, pad=0.1),
    "rand130_w7_deg16": dict(kind="rand", n=130, w=7, seed=6, deg=16, ia=20, pad=0.3),
    "rand257_w33_deg12": dict(kind="rand", n=257, w=33, seed=9, deg=12, ia=40, pad=0.2),
    # test_chfsi.py:101-108 — sigma scaling keeps degree 120 finite
    "rand40_w5_deg120": dict(kind="rand", n=40, w=5, seed=10, deg=120, ia=10, pad=1.0),
}


def build_filter_case(spec):
    rng = np.random.default_rng(spec["seed"])
    h = random_hermitian(rng, spec["n"])
    w, v = np.linalg.eigh(h)
    if spec["kind"] == "eig":
        return h, v, (float(w[20]), float(w[-1]) + 0.5, float(w[0])), spec["deg"]
    y = cgauss(rng, spec["n"], spec["w"])
    win = (float(w[spec["ia"]]), float(w[-1]) + spec["pad"], float(w[0]))
    return h, y, win, spec["deg"]


# ----------------------------------------------------------------- lanczos ---
LANCZOS_CASES = {
    **{f"rand100_k30_s{s}": dict(kind="rand", n=100, k=30, seed=s) for s in range(4)},
    "rand257_k51": dict(kind="rand", n=257, k=51, seed=21),
    "zero6_k4": dict(kind="zero", n=6, k=4, seed=0),        # test_chfsi.py:47-48
    "diag10_k10": dict(kind="diag", n=10, k=10, seed=3),    # test_chfsi.py:50-53
}


def build_lanczos_case(spec):
    n = spec["n"]
    if spec["kind"] == "zero":
        h = np.zeros((n, n), dtype=np.complex128)
    elif spec["kind"] == "diag":
        h = np.diag(np.arange(1.0, n + 1.0)).astype(np.complex128)
    else:
        h = random_hermitian(np.random.default_rng(spec["seed"]), n)
    return h, spec["k"], spec["seed"] + 100


# ---------------------------------------------------------------------- qr ---
QR_CASES = {
    "rand40x8": dict(kind="rand", m=40, n=8, seed=1),
    "rand203x37": dict(kind="rand", m=203, n=37, seed=2),
    "dup_col30x6": dict(kind="dup", m=30, n=6, seed=3),
    "zero_col20x4": dict(kind="zero", m=20, n=4, seed=4),
}


def build_qr_case(spec):
    rng = np.random.default_rng(spec["seed"])
    y = cgauss(rng, spec["m"], spec["n"])
    if spec["kind"] == "dup":
        y[:, 3] = y[:, 1]
    elif spec["kind"] == "zero":
        y[:, 2] = 0
    return y


# --------------------------------------------------------------- reduction ---
REDUCTION_CASES = {
    "pencil40": dict(kind="rand", n=40, seed=11, nv=5),
    "pencil131": dict(kind="rand", n=131, seed=12, nv=9),
    "diag_hand": dict(kind="hand"),                          # test_reduction.py:43-47
}


def build_reduction_case(spec):
    if spec["kind"] == "hand":
        a = np.diag([1.0, 2.0]).astype(np.complex128)
        b = np.diag([4.0, 1.0]).astype(np.complex128)
        return a, b, np.eye(2, dtype=np.complex128)
    rng = np.random.default_rng(spec["seed"])
    a = random_hermitian(rng, spec["n"])
    b = random_spd(rng, spec["n"], 100.0)
    y = cgauss(rng, spec["n"], spec["nv"])
    return a, b, y


# ------------------------------------------------------------------- solve ---
SOLVE_CASES = {
    # test_chfsi.py:137-143
    "diag100": dict(kind="diag", n=100, cfg=dict(nev=5, blk=12), seed=7),
    # test_chfsi.py:159-167
    "rand300_nev30": dict(kind="rand", n=300, hseed=1234, cfg=dict(nev=30), seed=11),
    # test_chfsi.py:169-187
    "rand90_accounting": dict(kind="rand", n=90, hseed=90, cfg=dict(nev=8, blk=20, deg=17), seed=2),
    # test_chfsi.py:189-195
    "rand120_nev10": dict(kind="rand", n=120, hseed=120, cfg=dict(nev=10, blk=26), seed=3),
    # test_chfsi.py:145-157
    "warm_exact80": dict(kind="warm", n=80, hseed=80, cfg=dict(nev=6), seed=5),
    # test_chfsi.py:218-225
    "partial_cap60": dict(kind="rand", n=60, hseed=60,
                          cfg=dict(nev=6, blk=14, max_repeats=1, deg=2), seed=4),
    # test_chfsi.py:234-241
    "rand70_det": dict(kind="rand", n=70, hseed=70, cfg=dict(nev=5, blk=15), seed=42),
    # ragged sizes (not tile multiples)
    "rand200_ragged": dict(kind="rand", n=200, hseed=200, cfg=dict(nev=13, blk=21, deg=9), seed=8),
}


def build_solve_case(spec):
    n = spec["n"]
    if spec["kind"] == "diag":
        h = np.diag(np.arange(1.0, n + 1.0)).astype(np.complex128)
        return h, dict(spec["cfg"]), None, spec["seed"]
    h = random_hermitian(np.random.default_rng(spec["hseed"]), n)
    guess = None
    if spec["kind"] == "warm":
        w, v = np.linalg.eigh(h)
        nev = spec["cfg"]["nev"]
        blk = spec["cfg"].get("blk") or nev + 40
        blk = min(blk, n)
        guess = (v[:, :blk], float(w[0]), float(w[blk]))
    return h, dict(spec["cfg"]), guess, spec["seed"]
