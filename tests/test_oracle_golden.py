"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The fixtures were produced by running the unmodified reference
(`tests/golden/make_golden.py`); these tests prove the numpy restatement in
`oracle/chfsi_oracle.py` reproduces them — counts exactly, floating-point
results to ~1e-12 — before the oracle is trusted as the checker of the
device path.
"""

import numpy as np
import pytest

from oracle import chfsi_oracle as orc
from paper_1206_3768_b200.sequence import BASELINE_CONFIGS, iter_baseline_sequence
from tests.conftest import subspace_sines
from tests.golden.recipes import (
    FILTER_CASES,
    LANCZOS_CASES,
    QR_CASES,
    REDUCTION_CASES,
    SOLVE_CASES,
    build_filter_case,
    build_lanczos_case,
    build_qr_case,
    build_reduction_case,
    build_solve_case,
    sha,
)


@pytest.mark.parametrize("name", sorted(FILTER_CASES))
def test_filter_matches_reference(small_golden, name):
    h, y, (a, b, s), deg = build_filter_case(FILTER_CASES[name])
    assert sha(h) == small_golden[f"filter/{name}/h_sha"].item().decode()
    assert sha(y) == small_golden[f"filter/{name}/y_sha"].item().decode()
    ref = small_golden[f"filter/{name}/out"]
    out = orc.chebyshev_filter(h, y, deg, a, b, s)
    assert np.abs(out - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())
    lam = np.linspace(s, b + 0.5, 41)
    np.testing.assert_allclose(orc.chebyshev_response(lam, deg, a, b, s),
                               small_golden[f"filter/{name}/response"], rtol=1e-13, atol=0)


@pytest.mark.parametrize("name", sorted(LANCZOS_CASES))
def test_lanczos_matches_reference(small_golden, name):
    h, k, seed = build_lanczos_case(LANCZOS_CASES[name])
    ritz, last, steps = orc.lanczos(h, k, np.random.default_rng(seed))
    assert steps == int(small_golden[f"lanczos/{name}/steps"])
    np.testing.assert_allclose(ritz, small_golden[f"lanczos/{name}/ritz"], rtol=0, atol=1e-12)
    assert abs(last - float(small_golden[f"lanczos/{name}/beta_last"])) <= 1e-12
    bound = float(ritz[-1] + last)
    assert abs(bound - float(small_golden[f"lanczos/{name}/bound"])) <= 1e-12


@pytest.mark.parametrize("name", sorted(QR_CASES))
def test_qr_matches_reference(small_golden, name):
    y = build_qr_case(QR_CASES[name])
    dead = small_golden[f"qr/{name}/dead"]
    if dead.size:
        with pytest.raises(orc.OracleRankDeficient) as err:
            orc.qr_orthonormalize(y)
        assert list(err.value.indices) == dead.tolist()
    else:
        q = orc.qr_orthonormalize(y)
        np.testing.assert_allclose(q, small_golden[f"qr/{name}/q"], rtol=0, atol=1e-13)


@pytest.mark.parametrize("name", sorted(REDUCTION_CASES))
def test_reduction_matches_reference(small_golden, name):
    a, b, y = build_reduction_case(REDUCTION_CASES[name])
    h, l = orc.to_standard(a, b)
    np.testing.assert_allclose(h, small_golden[f"reduction/{name}/h"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(l, small_golden[f"reduction/{name}/l"], rtol=0, atol=1e-13)
    x = orc.back_transform(l, y)
    np.testing.assert_allclose(x, small_golden[f"reduction/{name}/x"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", sorted(SOLVE_CASES))
def test_solve_matches_reference(small_golden, name):
    h, cfg, guess, seed = build_solve_case(SOLVE_CASES[name])
    vals, vecs, rep = orc.chfsi_solve(h, guess=guess, rng=np.random.default_rng(seed), **cfg)
    pre = f"solve/{name}/"
    assert rep.inner_loops == int(small_golden[pre + "inner_loops"])
    assert rep.matvecs == int(small_golden[pre + "matvecs"])
    assert rep.filtered_vectors == int(small_golden[pre + "filtered_vectors"])
    assert rep.lanczos_matvecs == int(small_golden[pre + "lanczos_matvecs"])
    assert rep.locked_per_loop == small_golden[pre + "locked_per_loop"].tolist()
    assert rep.converged == bool(small_golden[pre + "converged"])
    ref_vals = small_golden[pre + "values"]
    assert vals.shape == ref_vals.shape
    np.testing.assert_allclose(vals, ref_vals, rtol=0, atol=1e-12)
    if vals.size:
        assert subspace_sines(small_golden[pre + "vectors"], vecs).max() <= 1e-9


def test_c1_generator_bytes_and_harness_protocol(c1_golden):
    """BASELINE generator bytes + reference harness protocol on C1 (n=512)."""
    cfg = BASELINE_CONFIGS["C1"]
    prev = None
    for label, a, b in iter_baseline_sequence(cfg.n, cfg.length, seed=0):
        assert sha(a) == c1_golden[f"{label}/a_sha"].item().decode()
        assert sha(b) == c1_golden[f"{label}/b_sha"].item().decode()
        if label > 2:  # keep the CPU suite short: generator bytes for all, solves for 1-2
            continue
        h, l = orc.to_standard(a, b)
        assert sha(h) == c1_golden[f"{label}/h_sha"].item().decode()
        dv, dvec = orc.hermitian_eig(h)
        np.testing.assert_allclose(dv[: cfg.blk + 1], c1_golden[f"{label}/dense_values"],
                                   rtol=0, atol=1e-12)
        runs = [("cold", None, (0, label, 0))]
        if prev is not None:
            runs.append(("warm", prev, (0, label, 1)))
        for kind, guess, seed in runs:
            vals, vecs, rep = orc.chfsi_solve(h, cfg.nev, cfg.blk, cfg.deg, cfg.tol, guess=guess,
                                              rng=np.random.default_rng(seed))
            pre = f"{label}/{kind}/"
            assert rep.matvecs == int(c1_golden[pre + "matvecs"])
            assert rep.locked_per_loop == c1_golden[pre + "locked_per_loop"].tolist()
            np.testing.assert_allclose(vals, c1_golden[pre + "values"], rtol=0, atol=1e-12)
            assert subspace_sines(c1_golden[pre + "vectors"], vecs).max() <= 1e-9
        prev = (dvec[:, : cfg.blk], float(dv[0]), float(dv[cfg.blk]))


# ------------------------------------------------ adaptive degree (G4) ---
# No reference oracle exists for the adaptive mode: these pin the
# restatement's own invariants.

def test_adaptive_degree_rule():
    a, b, tol = 1.0, 9.0, 1e-10
    # converged -> floor; at/above the window edge -> cap; NaN -> cap
    assert orc.adaptive_degree(0.0, 1e-11, a, b, tol, 2, 36) == 2
    assert orc.adaptive_degree(a, 1e-3, a, b, tol, 2, 36) == 36
    assert orc.adaptive_degree(float("nan"), 1e-3, a, b, tol, 2, 36) == 36
    # t = (lam - c)/e = -1.5 -> rho = 1.5 + sqrt(1.25); r/tol = 1e4
    lam = 5.0 - 1.5 * 4.0
    import math
    d = math.ceil(math.log(1e4) / math.log(1.5 + math.sqrt(1.25))) + orc.ADAPTIVE_MARGIN
    assert orc.adaptive_degree(lam, 1e-6, a, b, tol, 2, 36) == d
    # monotone: a larger residual never asks for a lower degree
    ds = [orc.adaptive_degree(lam, r, a, b, tol, 2, 36) for r in (1e-9, 1e-7, 1e-5, 1e-3)]
    assert ds == sorted(ds)


def test_per_column_filter_is_the_definition():
    rng = np.random.default_rng(5)
    n, w = 40, 6
    g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = (g + g.conj().T) / 2
    y = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
    degs = [3, 1, 4, 1, 5, 2]
    out = orc.chebyshev_filter_degrees(h, y, degs, -1.0, 12.0, -3.0)
    for j, d in enumerate(degs):
        ref = orc.chebyshev_filter(h, y[:, j:j + 1], d, -1.0, 12.0, -3.0)
        # (BLAS may round a 1-column product differently from a 2-column one)
        assert np.abs(out[:, j:j + 1] - ref).max() <= 1e-13 * np.abs(ref).max()


def test_adaptive_solve_converges_with_fewer_flops_than_the_cap():
    """C1 shape: the adaptive mode reaches tol on every pair and spends
    less filter work than running every column at the cap."""
    from paper_1206_3768_b200.sequence import iter_baseline_sequence

    seq = list(iter_baseline_sequence(512, 3, seed=0))
    fixed = orc.run_sequence(seq, 32, 16, 24, adaptive=False)
    adapt = orc.run_sequence(seq, 32, 16, 24, adaptive=True)
    for f, a in zip(fixed, adapt):
        assert a["report"].converged
        assert a["report"].final_residuals.max() < 1e-10
        assert np.abs(a["values"] - f["values"]).max() <= 1e-9 * np.abs(f["values"]).max()
    assert sum(a["filter_flops"] for a in adapt) < sum(f["filter_flops"] for f in fixed)
