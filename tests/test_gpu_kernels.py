"""Device kernels vs the oracle and the reference golden vectors (B200 only).

Tolerances (floating point, the `north_star` bar is on eigenpairs; these
are the kernel-level bars that feed it):
* K1 / filter: max|out - ref| <= 1e-12 * max|ref| (the reference's own
  eigenbasis test uses 1e-12 * max|s|, test_chfsi.py:77);
* Lanczos Ritz values / bound: 1e-10 absolute on O(10) spectra;
* QR: 1e-12 (the positive-diagonal QR is unique);
* reduction H, L: 1e-12 * scale.
Integer results (Lanczos step counts, rank-deficient column indices) are
bit-exact.
"""

import ctypes

import numpy as np
import pytest
import torch

from oracle import chfsi_oracle as orc
from tests.golden.recipes import (
    FILTER_CASES,
    LANCZOS_CASES,
    QR_CASES,
    REDUCTION_CASES,
    build_filter_case,
    build_lanczos_case,
    build_qr_case,
    build_reduction_case,
    random_hermitian,
)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_1206_3768_b200 as p

    assert torch.cuda.is_available()
    return p


def _lib():
    from paper_1206_3768_b200 import _lib

    return _lib


def set_tiling(bm, bn, split, groups=1, warps=0):
    L = _lib()
    L.check(L.lib().chfsi_ctx_set_tiling(L.ctx(), bm, bn, split))
    if bm and groups != 1:
        L.check(L.lib().chfsi_ctx_set_step_groups(L.ctx(), groups))
    if bm and warps:
        L.check(L.lib().chfsi_ctx_set_step_warps(L.ctx(), warps))


@pytest.fixture(params=[3, 4], ids=["3m", "4m"])
def product(request):
    """K1 complex product: 3 = Gauss/3M (the default), 4 = four real MMAs."""
    L = _lib()
    old = L.lib().chfsi_set_complex_product(request.param)
    assert old in (3, 4)
    yield request.param
    L.lib().chfsi_set_complex_product(old)


# 3M-only variants: 32x16 warp tiles (4-warp 64-row, 8-warp 128-row CTAs)
TILINGS_3M = {(64, 32, 0, 1, 4), (64, 32, 7, 1, 4), (64, 16, 0, 1, 4), (64, 16, 13, 1, 4),
              (128, 32, 0, 1, 8), (128, 32, 5, 1, 8), (64, 32, 150, 1, 4)}


def cheb_step(h_dev, conj, ycur, yprev, ynext, alpha, c, beta):
    L = _lib()
    from paper_1206_3768_b200._device import ld_of

    n, w = ycur.shape
    ldh = h_dev.stride(0) if not conj else h_dev.stride(1)
    L.check(L.lib().chfsi_cheb_step_z(L.ctx(), n, w, L.dptr(h_dev), ldh, int(conj), L.dptr(ycur),
                                      ld_of(ycur), None if yprev is None else L.dptr(yprev),
                                      0 if yprev is None else ld_of(yprev), L.dptr(ynext),
                                      ld_of(ynext), alpha, c, beta))


def fb(x):
    from paper_1206_3768_b200._device import to_fblock

    return to_fblock(x, copy=True)


# (bm, bn, grid): grid 0 = every resident CTA; small grids force other
# data-parallel / stream-K splits and multi-peer fix-ups
TILINGS = [(64, 64, 0), (64, 32, 0), (64, 16, 0), (64, 64, 1), (64, 32, 7), (64, 16, 13),
           (64, 64, 150), (64, 32, 296), (128, 32, 0), (128, 32, 5), (128, 16, 0), (128, 16, 77),
           (64, 32, 0, 2), (64, 32, 9, 2), (64, 16, 0, 2), (64, 16, 31, 2)] + sorted(TILINGS_3M)


@pytest.mark.parametrize("tiling", TILINGS)
@pytest.mark.parametrize("n,w", [(64, 32), (131, 7), (257, 33), (512, 48), (1000, 97)])
@pytest.mark.parametrize("conj", [False, True])
def test_cheb_step_matches_numpy(pkg, product, tiling, n, w, conj):
    if tiling in TILINGS_3M and product == 4:
        pytest.skip("3M-only tile variant")
    if tiling[:2] in ((64, 64), (32, 32), (32, 64)) and product == 3:
        pytest.skip("4M-only tile variant (3M falls back to it)")
    rng = np.random.default_rng(n * 7 + w)
    h = random_hermitian(rng, n)
    y = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
    yp = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
    alpha, c, beta = 0.37, -0.81, 0.55
    ref = alpha * (h @ y - c * y) - beta * yp
    hd = torch.from_numpy(h).cuda()
    if conj:  # hand the kernel column-major storage of H
        hd = torch.from_numpy(np.asfortranarray(h)).cuda()
        hd = hd.t().contiguous().t()
    set_tiling(*tiling)
    try:
        yd, ypd = fb(y), fb(yp)
        cheb_step(hd, conj, yd, ypd, ypd, alpha, c, beta)  # in place over Yprev
        out = ypd.cpu().numpy()
    finally:
        set_tiling(0, 0, 0)
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()


def test_cheb_step_plain_product_and_determinism(pkg, product):
    rng = np.random.default_rng(3)
    n, w = 700, 45
    h = random_hermitian(rng, n)
    y = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
    hd, yd = torch.from_numpy(h).cuda(), fb(y)
    o1, o2 = fb(np.zeros((n, w), complex)), fb(np.zeros((n, w), complex))
    cheb_step(hd, False, yd, None, o1, 1.0, 0.0, 0.0)
    cheb_step(hd, False, yd, None, o2, 1.0, 0.0, 0.0)
    ref = h @ y
    assert np.abs(o1.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
    assert torch.equal(o1, o2)  # bitwise run-to-run


@pytest.mark.parametrize("n,w,grid,bm,groups", [
    (2048, 160, 0, 64, 1), (2048, 131, 0, 64, 1), (2048, 97, 0, 64, 1), (1500, 40, 37, 64, 1),
    (700, 33, 0, 64, 1), (4096, 160, 0, 64, 1), (2048, 160, 0, 128, 1), (3000, 70, 0, 128, 1),
    (2048, 160, 0, 64, 2), (1500, 40, 37, 64, 2), (3000, 131, 0, 64, 2),
    (2048, 160, 0, 64, -4), (2048, 97, 0, 64, -4), (1500, 40, 37, 64, -4), (5000, 250, 0, 128, -8)])
def test_cheb_step_bitwise_repeatable(pkg, n, w, grid, bm, groups):
    """Stream-K fix-ups, TMA/mbarrier pipeline and warp convergence: 40
    back-to-back filters must agree bit for bit. (This caught two real
    races: divergent lanes entering mma.sync.aligned, and the missing
    generic->async proxy fence before releasing a TMA stage.)"""
    rng = np.random.default_rng(n + w)
    h = torch.from_numpy(random_hermitian(rng, n)).cuda()
    y = fb(rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w)))
    win = pkg.FilterWindow(a=-1.0, b=1.5, scale_ref=-1.6)
    # groups < 0: one group of -groups warps (the 3M 32x16-warp-tile kernels)
    set_tiling(bm, 32, grid, max(groups, 1), -groups if groups < 0 else 0)
    try:
        outs = [pkg.chebyshev_filter(h, y, 4, win) for _ in range(40)]
    finally:
        set_tiling(0, 0, 0)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("n,w", [(512, 48), (1000, 97), (2048, 160), (2048, 64), (3000, 123),
                                 (5000, 250)])
def test_two_chain_filter_matches_one_chain_and_oracle(pkg, n, w):
    """The default filter runs balanced column halves as two concurrent
    launch chains: same result as one chain (to rounding) and as the oracle,
    bitwise reproducible run to run."""
    L = _lib()
    rng = np.random.default_rng(n + w)
    h = random_hermitian(rng, n)
    y = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
    hd, yd = torch.from_numpy(h).cuda(), fb(y)
    ev = np.linalg.eigvalsh(h)
    win = pkg.FilterWindow(a=float(ev[n // 4]), b=float(ev[-1]) + 0.1, scale_ref=float(ev[0]))
    two = [pkg.chebyshev_filter(hd, yd, 6, win) for _ in range(5)]
    try:
        L.check(L.lib().chfsi_ctx_set_filter_chains(L.ctx(), 1))
        one = pkg.chebyshev_filter(hd, yd, 6, win)
    finally:
        L.check(L.lib().chfsi_ctx_set_filter_chains(L.ctx(), 2))
    for t in two[1:]:
        assert torch.equal(t, two[0])
    scale = one.abs().max().item()
    assert (two[0] - one).abs().max().item() <= 1e-13 * scale
    ref = orc.chebyshev_filter(h, y, 6, win.a, win.b, win.scale_ref)
    assert np.abs(two[0].cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("name", sorted(FILTER_CASES))
def test_filter_matches_reference_golden(pkg, small_golden, name):
    h, y, (a, b, s), deg = build_filter_case(FILTER_CASES[name])
    ref = small_golden[f"filter/{name}/out"]
    out = pkg.chebyshev_filter(h, y, deg, pkg.FilterWindow(a=a, b=b, scale_ref=s))
    got = out.cpu().numpy()
    assert np.isfinite(got).all()
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_filter_input_untouched_and_column_major_operator(pkg):
    h, y, (a, b, s), deg = build_filter_case(FILTER_CASES["rand257_w33_deg12"])
    yd = fb(y)
    keep = yd.clone()
    win = pkg.FilterWindow(a=a, b=b, scale_ref=s)
    out_row = pkg.chebyshev_filter(torch.from_numpy(h).cuda(), yd, deg, win)
    hcol = torch.from_numpy(h).cuda().t().contiguous().t()  # column-major storage
    out_col = pkg.chebyshev_filter(hcol, yd, deg, win)
    assert torch.equal(yd, keep)
    ref = orc.chebyshev_filter(h, y, deg, a, b, s)
    for out in (out_row, out_col):
        assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("n,w,degs,conj", [
    (257, 9, [3, 1, 4, 1, 5, 9, 2, 6, 5], False),      # unsorted: the API sorts and restores
    (512, 40, list(range(1, 41)), True),              # one column retires per step
    (1000, 97, [7] * 50 + [12] * 47, False),          # two groups, parities differ
    (300, 5, [4, 4, 4, 4, 4], False)])                # uniform == the fixed-degree filter
def test_filter_per_column_degrees(pkg, n, w, degs, conj):
    """Adaptive-degree filter: column j equals the degree-degs[j]
    filter of y[:, j] (oracle: chebyshev_filter_degrees)."""
    rng = np.random.default_rng(n + w)
    h = random_hermitian(rng, n)
    y = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
    ev = np.linalg.eigvalsh(h)
    a, b, s = float(ev[n // 3]), float(ev[-1]) + 0.1, float(ev[0])
    hd = torch.from_numpy(h).cuda()
    if conj:
        hd = hd.t().contiguous().t()
    out = pkg.chebyshev_filter(hd, fb(y), degs, pkg.FilterWindow(a=a, b=b, scale_ref=s)).cpu().numpy()
    ref = orc.chebyshev_filter_degrees(h, y, degs, a, b, s)
    for j in range(w):  # per column: the degrees differ in scale by orders of magnitude
        assert np.abs(out[:, j] - ref[:, j]).max() <= 1e-12 * np.abs(ref[:, j]).max(), j
    if len(set(degs)) == 1:
        fixed = pkg.chebyshev_filter(hd, fb(y), degs[0], pkg.FilterWindow(a=a, b=b, scale_ref=s))
        assert np.abs(fixed.cpu().numpy() - out).max() <= 1e-13 * np.abs(out).max()


def test_filter_per_column_degrees_rejects_bad_input(pkg):
    h = torch.eye(16, dtype=torch.complex128, device="cuda")
    y = fb(np.ones((16, 3), dtype=complex))
    win = pkg.FilterWindow(a=0.5, b=2.0, scale_ref=-1.0)
    with pytest.raises(ValueError):
        pkg.chebyshev_filter(h, y, [1, 0, 2], win)
    with pytest.raises(ValueError):
        pkg.chebyshev_filter(h, y, [1, 2], win)


@pytest.mark.parametrize("name", sorted(LANCZOS_CASES))
def test_lanczos_matches_reference_golden(pkg, small_golden, name):
    from paper_1206_3768_b200.chfsi import _lanczos_estimates
    from paper_1206_3768_b200._device import Operator

    h, k, seed = build_lanczos_case(LANCZOS_CASES[name])
    ritz, last, steps = _lanczos_estimates(Operator(h), k, np.random.default_rng(seed))
    assert steps == int(small_golden[f"lanczos/{name}/steps"])
    np.testing.assert_allclose(ritz, small_golden[f"lanczos/{name}/ritz"], rtol=0, atol=1e-10)
    bound = pkg.lanczos_upper_bound(h, k, rng=np.random.default_rng(seed))
    assert abs(bound - float(small_golden[f"lanczos/{name}/bound"])) <= 1e-10


@pytest.mark.parametrize("n,k", [(2048, 204), (777, 60), (300, 300)])
def test_lanczos_cooperative_matches_multikernel(pkg, n, k):
    """The single cooperative kernel and the one-launch-per-operation path
    run the same algorithm: same step count, Ritz values to rounding."""
    from paper_1206_3768_b200.chfsi import _lanczos_estimates
    from paper_1206_3768_b200._device import Operator

    L = _lib()
    h = random_hermitian(np.random.default_rng(n), n)
    op = Operator(h)
    runs = {}
    try:
        for mode in (1, 0, 0):
            L.check(L.lib().chfsi_ctx_set_lanczos_mode(L.ctx(), mode))
            runs.setdefault(mode, []).append(_lanczos_estimates(op, k, np.random.default_rng(9)))
    finally:
        L.check(L.lib().chfsi_ctx_set_lanczos_mode(L.ctx(), 0))
    (r1, b1, s1), = runs[1]
    (r0, b0, s0), (r0b, b0b, s0b) = runs[0]
    assert s0 == s1 == s0b
    np.testing.assert_allclose(r0, r1, rtol=0, atol=1e-11)
    assert abs(b0 - b1) <= 1e-11
    assert np.array_equal(r0, r0b) and b0 == b0b  # bitwise run to run
    ritz_np, last_np, steps_np = orc.lanczos(h, k, np.random.default_rng(9))
    assert steps_np == s0
    np.testing.assert_allclose(r0, ritz_np, rtol=0, atol=1e-10)


def test_lanczos_rejects_too_few_steps(pkg):
    with pytest.raises(ValueError):
        pkg.lanczos_upper_bound(np.eye(3, dtype=complex), 1)


@pytest.mark.parametrize("name", sorted(QR_CASES))
def test_qr_matches_reference_golden(pkg, small_golden, name):
    y = build_qr_case(QR_CASES[name])
    dead = small_golden[f"qr/{name}/dead"]
    if dead.size:
        with pytest.raises(pkg.RankDeficientError) as err:
            pkg.qr_orthonormalize(y)
        assert list(err.value.indices) == dead.tolist()
    else:
        q = pkg.qr_orthonormalize(y).cpu().numpy()
        np.testing.assert_allclose(q, small_golden[f"qr/{name}/q"], rtol=0, atol=1e-12)


def set_qr_mode(mode):
    L = _lib()
    L.check(L.lib().chfsi_ctx_set_qr_mode(L.ctx(), mode))


@pytest.mark.parametrize("mode", [0, 2])
@pytest.mark.parametrize("kind", ["random", "graded", "near_dependent", "tall"])
def test_cholqr3_matches_householder(pkg, kind, mode):
    """Cholesky-QR2 with its shifted-QR3 escalation (mode 0, default) and
    shifted Cholesky-QR3 (mode 2) vs Householder: the same unique Q
    (positive-real R diagonal) to rounding x cond, orthonormal to 1e-13."""
    rng = np.random.default_rng(31)
    m, n = (4000, 24) if kind == "tall" else (300, 40)
    y = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    cond = 1.0
    if kind == "graded":  # filtered-panel-like column scales down to 1e-9
        y = y * np.logspace(0, -9, n)
        cond = 1e9
    elif kind == "near_dependent":
        y[:, 7] = y[:, 3] + 1e-8 * y[:, 7]
        cond = 1e8
    try:
        set_qr_mode(1)
        qh = pkg.qr_orthonormalize(y).cpu().numpy()
        set_qr_mode(mode)
        qc = pkg.qr_orthonormalize(y).cpu().numpy()
    finally:
        set_qr_mode(0)
    assert np.abs(qc.conj().T @ qc - np.eye(n)).max() <= 1e-13
    assert np.abs(qc - qh).max() <= 1e-13 * cond * 10
    ref = orc.qr_orthonormalize(y)
    assert np.abs(qc - ref).max() <= 1e-13 * cond * 10


@pytest.mark.parametrize("kind", ["random", "moderate", "graded", "tall_wide", "herk_trmm"])
def test_cholqr2_linearised_second_pass(pkg, kind):
    """Cholesky-QR2's linearised second pass (Q = Q1 (I - tri(Q1^H Q1 - I)),
    taken when the first pass leaves |Q1^H Q1 - I| <= 1e-8; the graded panel
    (cond 1e9) exceeds that and reruns the exact pass): same Q as the exact
    pass and as Householder to rounding x cond, orthonormal to 1e-13."""
    L = _lib()
    rng = np.random.default_rng(77)
    # herk_trmm: w >= 1000 takes the ZHERK Gram and the out-of-place ZTRMM
    m, n = {"tall_wide": (2048, 160), "herk_trmm": (2500, 1024)}.get(kind, (600, 48))
    y = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    cond = 1.0
    if kind == "moderate":  # the filtered panels' regime: R diagonal ranging over ~50
        y = y * np.logspace(0, -1.7, n)
        cond = 50.0
    elif kind == "graded":
        y = y * np.logspace(0, -9, n)
        cond = 1e9
    try:
        L.check(L.lib().chfsi_ctx_set_qr_linear2(L.ctx(), 0))
        q_exact = pkg.qr_orthonormalize(y).cpu().numpy()
        L.check(L.lib().chfsi_ctx_set_qr_linear2(L.ctx(), 1))
        q_lin = pkg.qr_orthonormalize(y).cpu().numpy()
        set_qr_mode(1)
        qh = pkg.qr_orthonormalize(y).cpu().numpy()
    finally:
        set_qr_mode(0)
        L.check(L.lib().chfsi_ctx_set_qr_linear2(L.ctx(), 1))
    assert np.abs(q_lin.conj().T @ q_lin - np.eye(n)).max() <= 1e-13
    assert np.abs(q_lin - q_exact).max() <= 1e-13 * cond * 10
    assert np.abs(q_lin - qh).max() <= 1e-13 * cond * 10


def test_qr_idempotent_on_orthonormal_input(pkg):
    rng = np.random.default_rng(17)
    q0 = orc.qr_orthonormalize(rng.standard_normal((90, 12)) + 1j * rng.standard_normal((90, 12)))
    q = pkg.qr_orthonormalize(q0).cpu().numpy()
    assert np.abs(q - q0).max() <= 1e-13


@pytest.mark.parametrize("n", [1, 7, 48, 160, 301])
def test_hermitian_eig(pkg, n):
    rng = np.random.default_rng(n)
    g = random_hermitian(rng, n)
    vals, vecs = pkg.hermitian_eig(g)
    np.testing.assert_allclose(vals, np.linalg.eigvalsh(g), rtol=0, atol=1e-12 * max(1, n))
    v = vecs.cpu().numpy()
    assert np.abs(v.conj().T @ v - np.eye(n)).max() <= 1e-12 * max(1, n)
    assert np.abs(g @ v - v * vals).max() <= 1e-11 * max(1, n)


@pytest.mark.parametrize("n,off", [(48, 1e-4), (160, 1e-6), (301, 1e-5), (160, 0.3), (37, 1e-5),
                                   (123, 1e-4), (256, 1e-6), (2, 1e-6), (9, 1e-3)])
def test_near_diagonal_eigensolver(pkg, n, off):
    """chfsi_heev_rr_z: near-diagonal G (the RR regime after the first loops)
    goes through the Jacobi/DMMA path (one cooperative kernel for n <= 256,
    ragged n included; the multi-kernel ZGEMM version above); a
    far-from-diagonal G must fall back
    to zheevd. Either way: ascending values and an orthonormal eigenbasis
    matching numpy to rounding."""
    from paper_1206_3768_b200._device import to_fblock, ld_of

    L = _lib()
    rng = np.random.default_rng(n)
    d = np.sort(rng.uniform(-1, 9, n))
    e = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * off
    g = np.diag(d) + (e + e.conj().T) / 2
    gd = to_fblock(g, copy=True)
    w = torch.empty(n, dtype=torch.float64, device="cuda")
    used = ctypes.c_int()
    L.check(L.lib().chfsi_heev_rr_z(L.ctx(), n, L.dptr(gd), ld_of(gd), L.dptr(w), 1e-13,
                                    ctypes.byref(used)))
    if off >= 0.1:
        assert used.value == 0      # far from diagonal: zheevd
    elif off <= 1e-5:
        assert used.value == 1      # clearly near-diagonal: the Jacobi/ZGEMM path
    vals, v = w.cpu().numpy(), gd.cpu().numpy()
    ref = np.linalg.eigvalsh(g)
    assert np.all(np.diff(vals) >= 0)
    np.testing.assert_allclose(vals, ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    assert np.abs(v.conj().T @ v - np.eye(n)).max() <= 1e-12
    assert np.abs(g @ v - v * vals).max() <= 1e-12 * np.abs(ref).max()


def test_hermitian_view_rejects_asymmetric(pkg):
    rng = np.random.default_rng(5)
    m = rng.standard_normal((6, 6)) + 1j * rng.standard_normal((6, 6))
    with pytest.raises(pkg.NotHermitianError):
        pkg.hermitian_view(m)
    h = random_hermitian(rng, 5)
    h[0, 1] += 1e-6
    with pytest.raises(pkg.NotHermitianError):
        pkg.hermitian_view(h, tol=1e-8)
    pkg.hermitian_view(h, tol=1e-3)


@pytest.mark.parametrize("name", sorted(REDUCTION_CASES))
def test_reduction_matches_reference_golden(pkg, small_golden, name):
    a, b, y = build_reduction_case(REDUCTION_CASES[name])
    sp = pkg.to_standard(pkg.EigenPencil(a=a, b=b))
    h = sp.h.cpu().numpy()
    l = sp.cholesky_factor.cpu().numpy()
    href = small_golden[f"reduction/{name}/h"]
    np.testing.assert_allclose(h, href, rtol=0, atol=1e-12 * max(1.0, np.abs(href).max()))
    assert np.array_equal(h, h.conj().T)  # exactly Hermitian after re-symmetrization
    np.testing.assert_allclose(l, small_golden[f"reduction/{name}/l"], rtol=0, atol=1e-12)
    sol = pkg.EigenSolution(values=np.zeros(y.shape[1]), vectors=y)
    x = pkg.back_transform(sp.cholesky_factor, sol).vectors.cpu().numpy()
    xref = small_golden[f"reduction/{name}/x"]
    np.testing.assert_allclose(x, xref, rtol=0, atol=1e-11 * max(1.0, np.abs(xref).max()))


@pytest.mark.parametrize("n,nev", [(100, 7), (256, 33), (700, 40), (1500, 97), (2048, 128)])
def test_back_transform_blocked_matches_triangular_solve(pkg, n, nev):
    """x = L^-H y through the backward block substitution (K1 products with
    the rows of L^H right of the diagonal, ZTRSM on the 256-row diagonal
    blocks) vs scipy's triangular solve."""
    import scipy.linalg

    rng = np.random.default_rng(n)
    c = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    b = np.eye(n) + c @ c.conj().T / (4 * n)
    l = np.linalg.cholesky(b)
    y = rng.standard_normal((n, nev)) + 1j * rng.standard_normal((n, nev))
    sol = pkg.EigenSolution(values=np.zeros(nev), vectors=y)
    x = pkg.back_transform(torch.from_numpy(np.asfortranarray(l)).cuda().t().contiguous().t(),
                           sol).vectors.cpu().numpy()
    ref = scipy.linalg.solve_triangular(l, y, lower=True, trans="C")
    assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("n", [64, 255, 256, 700, 1100])
def test_to_standard_k1_matches_numpy(pkg, n):
    """The sequence driver's reduction (chfsi_to_standard_k1_z: block
    substitutions with K1 products) vs numpy's L^-1 A L^-H, and vs the
    ZTRSM path of to_standard()."""
    import scipy.linalg
    from paper_1206_3768_b200.reduction import stage_standard

    rng = np.random.default_rng(n + 3)
    a = random_hermitian(rng, n)
    c = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    b = np.eye(n) + c @ c.conj().T / (4 * n)
    l = np.linalg.cholesky(b)
    z = scipy.linalg.solve_triangular(l, a, lower=True)
    href = scipy.linalg.solve_triangular(l, z.conj().T, lower=True)
    href = (href + href.conj().T) / 2
    _, sp, checks = stage_standard(a, b, 1)
    torch.cuda.synchronize()
    checks.raise_if_invalid()
    h = sp.h.cpu().numpy()
    assert np.array_equal(h, h.conj().T)
    assert np.abs(h - href).max() <= 1e-12 * np.abs(href).max()
    assert np.abs(sp.cholesky_factor.cpu().numpy() - l).max() <= 1e-12
    h_trsm = pkg.to_standard(pkg.EigenPencil(a=a, b=b)).h.cpu().numpy()
    assert np.abs(h - h_trsm).max() <= 1e-13 * np.abs(href).max()


def test_reduction_rejects_indefinite_overlap(pkg):
    rng = np.random.default_rng(8)
    a = random_hermitian(rng, 6)
    b = random_hermitian(rng, 6)
    with pytest.raises(pkg.NotPositiveDefiniteError):
        pkg.to_standard(pkg.EigenPencil(a=a, b=b))


def test_reduction_identity_overlap_is_noop(pkg):
    rng = np.random.default_rng(9)
    a = random_hermitian(rng, 7)
    sp = pkg.to_standard(pkg.EigenPencil(a=a, b=np.eye(7)))
    np.testing.assert_array_equal(sp.h.cpu().numpy(), a)


def test_symmetrize_and_defect_kernels(pkg):
    L = _lib()
    rng = np.random.default_rng(10)
    n = 77
    m = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    d = fb(m)
    L.check(L.lib().chfsi_symmetrize_z(L.ctx(), n, L.dptr(d), n))
    np.testing.assert_array_equal(d.cpu().numpy(), (m + m.conj().T) / 2)
    defect, scale = pkg.linalg.hermitian_defect(m)
    assert defect == pytest.approx(np.abs(m - m.conj().T).max(), rel=1e-15)
    assert scale == pytest.approx(np.abs(m).max(), rel=1e-15)


@pytest.mark.parametrize("m,n", [(512, 48), (2048, 160), (2048, 34), (2050, 101), (1000, 192), (300, 16),
                                 (77, 5)])
@pytest.mark.parametrize("mode", [0, 2])
def test_panel_kernels_match_library_qr(pkg, m, n, mode):
    """Cholesky-QR2 (mode 0: exact first pass + linearised second; mode 2:
    shifted three-pass) with the hand-written panel kernels (Y L^-H and the
    near-identity pass, panel_kernels.cu) vs the cuBLAS ZTRSM / ZGEMM chains:
    the same unique Q to rounding, orthonormal to 1e-13, bitwise repeatable;
    also against the oracle's Householder QR."""
    L = _lib()
    rng = np.random.default_rng(1000 * m + n)
    y = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    y = y * np.logspace(0, -1.5, n)  # filtered-panel-like column scales (cond ~ 30)
    prev = L.lib().chfsi_set_panel_kernels(-1)
    try:
        set_qr_mode(mode)
        L.lib().chfsi_set_panel_kernels(0)
        q_lib = pkg.qr_orthonormalize(y).cpu().numpy()
        L.lib().chfsi_set_panel_kernels(1)
        q_own = pkg.qr_orthonormalize(y).cpu().numpy()
        q_own2 = pkg.qr_orthonormalize(y).cpu().numpy()
    finally:
        set_qr_mode(0)
        L.lib().chfsi_set_panel_kernels(prev)
    assert np.array_equal(q_own, q_own2)
    assert np.abs(q_own.conj().T @ q_own - np.eye(n)).max() <= 1e-13
    assert np.abs(q_own - q_lib).max() <= 2e-12
    assert np.abs(q_own - orc.qr_orthonormalize(y)).max() <= 2e-12
