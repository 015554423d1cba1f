"""Synthetic correlated pencil sequences (the BASELINE.json generator).

The reference's own generator (`spectral_chain/sequence.py:137-178`) draws a
Gaussian Hermitian A and a log-spaced SPD B; BASELINE.json prescribes a
different recipe, restated here with a pinned draw order
so the CPU oracle and the device path see the SAME bytes:

* ``rng = numpy.random.default_rng(seed)``;
* complex standard Gaussian ``z = (N(0,1) + i N(0,1)) / sqrt(2)`` — the real
  block is drawn first, then the imaginary block;
* draw 1: ``C`` (n x n);   ``B1 = I + C C^H / (4n)``, re-symmetrized;
* draw 2: ``G`` (n x n);   ``Q, R = qr(G)``;  ``U = Q diag(conj(r_ii / |r_ii|))``
  (the phase fix of the reference test fixture `pkg/tests/conftest.py:19-22`);
* ``d_i = -1 + 11 (i/n)^1.5`` for ``i = 0..n-1``;  ``A1 = U diag(d) U^H``,
  re-symmetrized;
* for ``l = 1..N-1``: draw ``E_l`` then ``F_l``, each ``(G + G^H)/2`` of a fresh
  complex Gaussian rescaled to ``||.||_F = sqrt(n)``;
  ``eps_l = 1e-2 * 0.5**l``;  ``A_{l+1} = A_l + eps_l E_l``;
  ``B_{l+1} = B_l + (eps_l / 10) F_l``.

Problems are yielded lazily (``iter_baseline_sequence``) so that n=20000
sequences never hold more than one (A, B) pair plus the running sums.

``device=...`` keeps the host to what fixes the bytes'
distribution — the numpy Generator draws, in the same order — and does the
O(n^3) part on the GPU through libchfsi (ZGEMM for C C^H and U diag(d) U^H,
the positive-diagonal QR for the Haar U) plus the O(n^2) symmetrize /
rescale steps, yielding device tensors. Results equal the host generator's
to rounding (tests/test_gpu_io.py), and C5's generation drops from tens of
minutes of host LAPACK to the time of its random draws.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "CorrelationSchedule",
    "PencilSequence",
    "generate_sequence",
    "iter_generated_sequence",
    "BaselineConfig",
    "BASELINE_CONFIGS",
    "complex_gaussian",
    "hermitian_unit_frobenius",
    "iter_baseline_sequence",
    "generate_baseline_sequence",
]


@dataclass(frozen=True)
class BaselineConfig:
    """One row of BASELINE.json ``configs`` (SURVEY.md §8 shape table)."""

    name: str
    n: int
    length: int
    nev: int
    nex: int
    deg: int
    tol: float = 1e-10
    adaptive_degree: bool = False

    @property
    def blk(self) -> int:
        return self.nev + self.nex


BASELINE_CONFIGS = {
    "C1": BaselineConfig("C1", 512, 6, 32, 16, 12),
    "C2": BaselineConfig("C2", 2048, 10, 128, 32, 16),
    "C3": BaselineConfig("C3", 5000, 12, 500, 100, 20),
    "C4": BaselineConfig("C4", 12000, 8, 1200, 200, 20),
    "C5": BaselineConfig("C5", 20000, 6, 3000, 400, 36, adaptive_degree=True),
}


def complex_gaussian(rng, n, m):
    """i.i.d. complex standard Gaussian block (unit variance per entry)."""
    re = rng.standard_normal((n, m))
    im = rng.standard_normal((n, m))
    z = np.empty((n, m), dtype=np.complex128)
    z.real = re
    z.imag = im
    z *= 1.0 / np.sqrt(2.0)
    return z


def _symmetrize(m):
    return (m + m.conj().T) * 0.5


def hermitian_unit_frobenius(rng, n):
    """Hermitian Gaussian perturbation with ``||E||_F = sqrt(n)``."""
    g = complex_gaussian(rng, n, n)
    e = _symmetrize(g)
    e *= np.sqrt(n) / np.linalg.norm(e)
    return e


def iter_baseline_sequence(n, length, seed=0, device=None):
    """Yield ``(label, A_l, B_l)`` for l = 1..length (complex128, C-ordered).

    The yielded arrays are fresh copies; the generator keeps its own running
    ``A``/``B``. With ``device`` (e.g. ``"cuda:0"``) they are row-major CUDA
    tensors computed on the GPU from the same host draws.
    """
    if n < 2 or length < 1:
        raise ValueError("need n >= 2 and length >= 1")
    if device is not None:
        yield from _device_sequence(n, length, seed, device)
        return
    rng = np.random.default_rng(seed)
    c = complex_gaussian(rng, n, n)
    b = c @ c.conj().T
    b *= 1.0 / (4.0 * n)
    b[np.diag_indices(n)] += 1.0
    b = _symmetrize(b)
    del c
    g = complex_gaussian(rng, n, n)
    q, r = np.linalg.qr(g)
    del g
    rd = np.diagonal(r)
    u = q * (rd / np.abs(rd)).conj()
    del q, r
    d = -1.0 + 11.0 * (np.arange(n, dtype=np.float64) / n) ** 1.5
    a = (u * d) @ u.conj().T
    a = _symmetrize(a)
    del u
    yield 1, a.copy(), b.copy()
    for ell in range(1, length):
        eps = 1e-2 * 0.5**ell
        e = hermitian_unit_frobenius(rng, n)
        f = hermitian_unit_frobenius(rng, n)
        a += eps * e
        b += (eps / 10.0) * f
        del e, f
        yield ell + 1, a.copy(), b.copy()


def _device_sequence(n, length, seed, device):
    import torch

    from ._device import C128, fblock
    from ._lib import check, ctx, dptr, lib
    from .linalg import qr_orthonormalize_inplace

    dev = torch.device(device)

    def upload_gaussian():
        z = complex_gaussian(rng, n, n)
        return torch.from_numpy(z).pin_memory().to(dev, non_blocking=True)  # row-major

    def gemm_nc(x, y, alpha):  # alpha * x y^H for column-major n x n blocks
        out = fblock(n, n, dev)
        check(lib().chfsi_gemm_z(ctx(), b"N", b"C", n, n, n, alpha, 0.0, dptr(x), n, dptr(y), n,
                                 0.0, 0.0, dptr(out), n), "generator gemm")
        return out

    def symmetrize(m):  # column-major in place
        check(lib().chfsi_symmetrize_z(ctx(), n, dptr(m), n), "generator symmetrize")
        return m

    def herm_unit_frobenius():
        g = upload_gaussian()
        e = (g + g.conj().t()) * 0.5
        del g
        return e * (float(np.sqrt(n)) / torch.linalg.vector_norm(e).item())

    def colmajor(t):  # column-major copy of a (logical) n x n tensor
        return t.t().contiguous().t()

    rng = np.random.default_rng(seed)
    with torch.cuda.device(dev):
        c = colmajor(upload_gaussian())
        b = gemm_nc(c, c, 1.0 / (4.0 * n))        # C C^H / (4n)
        del c
        b.diagonal().add_(1.0)
        symmetrize(b)
        u = colmajor(upload_gaussian())
        qr_orthonormalize_inplace(u)              # Q diag(conj(r_ii/|r_ii|)): positive-real R
        d = torch.from_numpy(-1.0 + 11.0 * (np.arange(n, dtype=np.float64) / n) ** 1.5).to(dev)
        a = symmetrize(gemm_nc(u * d.to(C128)[None, :], u, 1.0))  # U diag(d) U^H
        del u
        a = a.contiguous()                        # row-major, like the host generator
        b = b.contiguous()
        yield 1, a.clone(), b.clone()
        for ell in range(1, length):
            eps = 1e-2 * 0.5**ell
            e = herm_unit_frobenius()
            f = herm_unit_frobenius()
            a.add_(e, alpha=eps)
            b.add_(f, alpha=eps / 10.0)
            del e, f
            yield ell + 1, a.clone(), b.clone()


def generate_baseline_sequence(n, length, seed=0):
    """Materialize the whole sequence as a list of ``(label, A, B)``."""
    return list(iter_baseline_sequence(n, length, seed))


# ------------------------------------------- the reference's own generator ---
# `run_experiment(ExperimentSpec(source=GenerateSource(...)))` feeds the
# reference generator (sequence.py:36-178), so that source is restated here
# with the same draw order; the arithmetic is numpy on the host like the
# reference's (it fixes the input bytes — np.linalg.qr's unphased Q is part
# of B), only the positive-definiteness probe of each B runs on the device
# (the library's potrf).

_EPS0, _DECAY = 0.5, 0.45  # geometric default, sequence.py:33-34


@dataclass
class CorrelationSchedule:
    """Perturbation magnitudes between adjacent problems
    (sequence.py:37-76): ``eps[i]`` takes problem i+1 to i+2 (A update),
    B is perturbed with eps/10 when ``perturb_b``."""

    length: int
    eps: list | None = None
    perturb_b: bool = True
    b_cond_target: float = 1e6

    def __post_init__(self):
        if self.length < 1:
            raise ValueError("a sequence has at least one problem")
        if self.eps is None:
            self.eps = [_EPS0 * _DECAY ** i for i in range(self.length - 1)]
        self.eps = [float(x) for x in self.eps]
        if len(self.eps) != self.length - 1:
            raise ValueError(f"need {self.length - 1} perturbation magnitudes, got {len(self.eps)}")
        if min(self.eps, default=0.0) < 0:
            raise ValueError("perturbation magnitudes must be non-negative")
        if self.b_cond_target < 1:
            raise ValueError("condition target must be >= 1")

    @classmethod
    def geometric(cls, length, eps0=_EPS0, decay=_DECAY, **kwargs):
        if eps0 <= 0 or not 0 < decay <= 1:
            raise ValueError("need eps0 > 0 and 0 < decay <= 1")
        return cls(length=length, eps=[eps0 * decay ** i for i in range(length - 1)], **kwargs)


@dataclass
class PencilSequence:
    """Pencils labelled 1..N of one dimension (sequence.py:79-101)."""

    pencils: list
    provenance: dict = field(default_factory=dict)

    def __post_init__(self):
        if not self.pencils:
            raise ValueError("empty sequence")
        n = self.pencils[0].n
        for pos, p in enumerate(self.pencils):
            if p.label != pos + 1:
                raise ValueError(f"labels must run 1..N, found {p.label} at position {pos}")
            if p.n != n:
                raise ValueError("all pencils must share one dimension")

    def __len__(self):
        return len(self.pencils)

    def __iter__(self):
        return iter(self.pencils)

    @property
    def n(self):
        return self.pencils[0].n


def _gaussian_hermitian(rng, n):
    """(G + G^H)/2 of G = (N + iN)/sqrt(2) (sequence.py:117-119)."""
    g = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2)
    return (g + g.conj().T) / 2


def _b_is_hpd(b):
    from .linalg import cholesky
    from .linalg_errors import NotPositiveDefiniteError

    try:
        cholesky(b)
    except NotPositiveDefiniteError:
        return False
    return True


def iter_generated_sequence(n, schedule, seed=None):
    """Lazily yield ``(label, A, B)`` host arrays of the reference generator
    (sequence.py:137-178, same draws in the same order): A1 Gaussian
    Hermitian, B1 = Q diag(logspace(0, log10 cond, n)) Q^H from the
    unphased QR of a complex Gaussian (sequence.py:127-134); then
    A += eps * D / max|D| and B += s * F / max|F| with s = eps/10 halved
    (up to 5 times) until B stays positive definite."""
    if n < 4:
        raise ValueError("need dimension >= 4")
    rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
    a = _gaussian_hermitian(rng, n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    spd = (q * np.logspace(0.0, np.log10(schedule.b_cond_target), n)) @ q.conj().T
    b = (spd + spd.conj().T) / 2
    del q, spd
    yield 1, a, b
    for i, eps in enumerate(schedule.eps):
        d = _gaussian_hermitian(rng, n)
        a = a + eps * (d / np.abs(d).max())
        if schedule.perturb_b:
            f = _gaussian_hermitian(rng, n)
            f = f / np.abs(f).max()
            scale = eps / 10
            for attempt in range(6):
                cand = b + scale * f
                if _b_is_hpd(cand):
                    break
                if attempt == 5:
                    from .linalg_errors import NotPositiveDefiniteError

                    raise NotPositiveDefiniteError(
                        f"overlap update {i + 1} breaks positive definiteness after 5 halvings")
                scale /= 2
            b = cand
        yield i + 2, a, b


def generate_sequence(n, schedule, seed=None):
    """The reference generator as a PencilSequence of device EigenPencils
    (sequence.py:137-178)."""
    from .reduction import EigenPencil

    pencils = [EigenPencil(a=a, b=b, label=lab)
               for lab, a, b in iter_generated_sequence(n, schedule, seed)]
    return PencilSequence(pencils=pencils, provenance={
        "kind": "generated", "n": n, "length": schedule.length, "eps": list(schedule.eps),
        "perturb_b": schedule.perturb_b, "b_cond_target": schedule.b_cond_target,
        "seed": None if isinstance(seed, np.random.Generator) else seed})
