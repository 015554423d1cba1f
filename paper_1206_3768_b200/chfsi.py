"""Chebyshev Filtered Subspace Iteration with locking — device path.

Drop-in for `spectral_chain.chfsi` (reference `chfsi.py:1-384`): same
names, signatures, counters and exceptions. Every operation on n-sized data
runs on the GPU through libchfsi:

* the filter (K1, `chfsi_filter_z`: one fused DMMA kernel per recurrence
  step, shift/scale/three-term update in the epilogue, ping-pong in place);
* the Lanczos bound (K2, `chfsi_lanczos_z`: HBM-bound GEMV + deterministic
  reorthogonalization, no host sync per step);
* CGS against the locked block and the Householder QR (K3);
* Rayleigh-Ritz (K4: H*panel through K1, cuBLAS Gram/rotations, cuSOLVER
  zheevd on the blk x blk projection, fused residual column norms).

Only O(blk) scalars cross to the host: the Ritz values and residual norms
that drive locking (chfsi.py:352-373), the k x k Lanczos tridiagonal, and
the random draws, which are made on the host with the caller's numpy
Generator in exactly the reference order so iteration counts match.
"""

from __future__ import annotations

import ctypes
import os
import threading
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import torch

from ._device import Operator, emit, fblock, host_output, ld_of, to_fblock, to_host
from ._lib import ALLREDUCE_CB, FILL_CB, FILTER_CB, GATHER_CB, HP_CB, LoopState, check, ctx, dptr, lib
from .linalg import qr_orthonormalize_inplace
from .reduction import EigenSolution

__all__ = [
    "ChfsiConfig",
    "FilterWindow",
    "ChfsiGuess",
    "SolveReport",
    "lanczos_upper_bound",
    "chebyshev_filter",
    "chebyshev_response",
    "rayleigh_ritz",
    "chfsi_solve",
    "filter_flops",
]


@dataclass
class ChfsiConfig:
    """Solver parameters (chfsi.py:36-69).

    ``blk`` defaults to ``nev + 40``; ``nex`` (BASELINE.json's name for the
    extra vectors) is accepted as an alias: ``blk = nev + nex``.
    ``adaptive_degree`` (additive, config C5 / SURVEY G4): per-vector filter
    degrees capped at ``deg`` and floored at ``min_degree``, chosen after
    every pass from each unlocked Ritz pair's residual (the rule is restated
    in oracle/chfsi_oracle.py). Off by default: the reference's fixed degree.
    """

    nev: int
    blk: int | None = None
    deg: int = 25
    tol: float = 1e-10
    lanczos_steps: int | None = None
    max_repeats: int = 50
    nex: int | None = None
    adaptive_degree: bool = False
    min_degree: int = 2

    def __post_init__(self):
        if self.nex is not None:
            if self.blk is not None and self.blk != self.nev + self.nex:
                raise ValueError("give either blk or nex, not conflicting values")
            self.blk = self.nev + self.nex

    def resolve(self, n):
        """Fill in size-dependent defaults and validate against ``n``."""
        blk = self.blk if self.blk is not None else self.nev + 40
        blk = min(blk, n)
        if not (1 <= self.nev <= blk <= n):
            raise ValueError(f"need 1 <= nev <= blk <= n, got nev={self.nev}, blk={blk}, n={n}")
        if self.deg < 1:
            raise ValueError("polynomial degree must be >= 1")
        if self.adaptive_degree and not 1 <= self.min_degree <= self.deg:
            raise ValueError("adaptive degree needs 1 <= min_degree <= deg")
        if self.tol <= 0:
            raise ValueError("tolerance must be positive")
        if self.lanczos_steps is not None:
            k = self.lanczos_steps
        else:
            k = min(3 * blk, max(10, n // 10))
            k = max(k, min(10, 3 * blk))
        k = max(2, min(k, n))
        return blk, self.deg, self.tol, k, self.max_repeats


@dataclass(frozen=True)
class FilterWindow:
    """Damped interval ``[a, b]`` and the growth anchor (chfsi.py:72-88)."""

    a: float
    b: float
    scale_ref: float

    def __post_init__(self):
        if not self.a < self.b:
            raise ValueError(f"need a < b, got a={self.a}, b={self.b}")
        if not self.scale_ref < self.a:
            raise ValueError(f"need scale_ref < a, got scale_ref={self.scale_ref}, a={self.a}")


@dataclass(frozen=True)
class ChfsiGuess:
    """Warm start (chfsi.py:91-98): ``blk`` vectors (numpy or device
    tensor) plus the previous lambda_1 and lambda_{blk+1}."""

    vectors: object
    lambda1: float
    lambda_blk_plus_1: float


@dataclass
class SolveReport:
    """Work counters of one solve (chfsi.py:101-122), same algebra:
    ``matvecs == deg*filtered_vectors + lanczos_matvecs + residual_check_matvecs``.

    Additive fields: device phase times (CUDA events, seconds), the filter
    FLOP count (8 n^2 per column per degree), and the chained-mode tail
    (the full final ``blk`` block and the largest final Ritz value, the
    lambda_{blk+1} proxy of SURVEY G2).
    """

    inner_loops: int = 0
    filtered_vectors: int = 0
    matvecs: int = 0
    lanczos_matvecs: int = 0
    residual_check_matvecs: int = 0
    locked_per_loop: list = field(default_factory=list)
    final_residuals: np.ndarray = field(default_factory=lambda: np.zeros(0))
    wall_time: float = 0.0
    converged: bool = False
    operator_norm_estimate: float = 0.0
    ritz_history: list = field(default_factory=list)
    t_lanczos: float = 0.0
    t_filter: float = 0.0
    t_ortho: float = 0.0
    t_rr: float = 0.0
    filter_flops: float = 0.0
    filter_launches: int = 0
    # K1 work the filter actually executed: from the second pass on its first
    # step reuses the previous Rayleigh-Ritz's H*P (elementwise, no product)
    filter_k1_flops: float = 0.0
    filter_k1_launches: int = 0
    rr_fast_eigs: int = 0
    qr_redone: int = 0  # passes whose speculative Cholesky-QR2 was redone on the full path
    filter_degree_sum: int = 0  # sum of per-column degrees (= deg * filtered_vectors unless adaptive)
    tail_vectors: object = None
    lambda_blk_plus_1: float = float("nan")
    host_phases: dict = field(default_factory=dict)  # wall seconds per host phase


def filter_flops(n, deg, columns):
    """Algorithmic FLOPs of the filter: 8 n^2 per column per degree."""
    return 8.0 * float(n) * float(n) * float(deg) * float(columns)


def as_rng(seed_or_rng):
    """Coerce None / int / tuple / Generator to a Generator (_util.py:8-12)."""
    if isinstance(seed_or_rng, np.random.Generator):
        return seed_or_rng
    return np.random.default_rng(seed_or_rng)


def _draw_block(rng, n, cols, pinned=False):
    """Complex Gaussian block drawn on the host in the reference order
    (_util.py:15-18: real parts, then imaginary parts, each C-ordered), as a
    CPU complex128 tensor, page-locked with ``pinned``. The two draws go
    through one float scratch straight into the complex storage: the same
    bytes as ``re + 1j * im`` without its complex temporaries (~3 ms less
    host time at C2) or a separate copy into page-locked memory."""
    out = torch.empty((n, cols), dtype=torch.complex128, pin_memory=pinned)
    z = out.numpy()
    tmp = np.empty((n, cols))
    rng.standard_normal(out=tmp)
    z.real = tmp
    rng.standard_normal(out=tmp)
    z.imag = tmp
    return out


class PrefetchedStart:
    """The cold-start draws of one solve — the Lanczos vector q0 (chfsi.py:137)
    then the (n, blk) start block (chfsi.py:323, _util.py:15-18) — taken from
    ``rng`` in that order on a host thread started ahead of the solve (the
    sequence driver starts it before problem 1's upload and reduction), the
    block staged in page-locked memory. Pass it as ``rng`` to chfsi_solve:
    later draws (rank repair) continue from the same generator, exactly as if
    the solve had drawn everything itself."""

    def __init__(self, rng, n, blk):
        self.rng, self.n, self.blk = as_rng(rng), n, blk
        self._q0_ready = threading.Event()
        self._box = {}
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()

    def _run(self):
        try:
            self._box["q0"] = _draw_start_vector(self.rng, self.n)
            self._q0_ready.set()
            self._box["z"] = _draw_block(self.rng, self.n, self.blk, pinned=True)
        except BaseException as exc:  # noqa: BLE001 - re-raised by the consumer
            self._box["err"] = exc
            self._q0_ready.set()

    def _check(self):
        if "err" in self._box:
            raise self._box["err"]

    def q0(self):
        self._q0_ready.wait()
        self._check()
        return self._box["q0"]

    def block(self):
        self._thread.join()
        self._check()
        return self._box["z"]


def random_block(rng, n, cols):
    """`_draw_block`, uploaded as a device F-block."""
    # page-locked staging: one DMA instead of a pageable copy (~10 ms at C2)
    return to_fblock(_draw_block(rng, n, cols, pinned=True))


class _PhaseTimer:
    """Accumulates device time of a phase with CUDA events on the launch stream."""

    def __init__(self):
        self.pairs = []

    def start(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.pairs.append([e, None])

    def stop(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.pairs[-1][1] = e

    def seconds(self):
        return sum(a.elapsed_time(b) for a, b in self.pairs if b is not None) / 1e3


# --------------------------------------------------------------- Lanczos ---

def _draw_start_vector(rng, n):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)  # chfsi.py:137 draw order


def _lanczos_estimates(op, k, rng, q0=None, comm=None):
    """k-step Lanczos with full reorthogonalization on the device
    (chfsi.py:125-162). Returns (ritz, beta_last, steps). ``q0``: the start
    vector when the caller already drew it; ``comm``: row-sharded over the
    ranks of a RowComm (same result on every rank)."""
    n = op.n
    k = min(k, n)
    if q0 is None:
        q0 = _draw_start_vector(rng, n)
    if comm is not None and comm.part.world > 1:
        from .distributed import lanczos_rows

        alphas, betas, beta_last, s = lanczos_rows(comm, op, k, q0)
        ritz = alphas[:1].copy() if s == 1 else scipy.linalg.eigvalsh_tridiagonal(alphas[:s],
                                                                                  betas[: s - 1])
        return ritz, beta_last, s
    q0d = torch.from_numpy(q0).to(op.tensor.device)
    basis = fblock(n, k)
    alphas = np.zeros(k)
    betas = np.zeros(k)
    beta_last = ctypes.c_double()
    steps = ctypes.c_int()
    pd = ctypes.POINTER(ctypes.c_double)
    check(lib().chfsi_lanczos_z(ctx(), n, k, dptr(op.tensor), op.ld, op.conj, dptr(q0d),
                                dptr(basis), alphas.ctypes.data_as(pd), betas.ctypes.data_as(pd),
                                ctypes.byref(beta_last), ctypes.byref(steps)), "lanczos")
    s = steps.value
    if s == 1:
        ritz = alphas[:1].copy()
    else:
        ritz = scipy.linalg.eigvalsh_tridiagonal(alphas[:s], betas[: s - 1])
    return ritz, beta_last.value, s


def lanczos_upper_bound(h, k, rng=None):
    """Largest Ritz value plus the final residual norm (chfsi.py:165-176)."""
    if k < 2:
        raise ValueError("need at least 2 Lanczos steps")
    ritz, beta_last, _ = _lanczos_estimates(Operator.wrap(h), k, as_rng(rng))
    return float(ritz[-1] + beta_last)


# ---------------------------------------------------------------- filter ---

def _filter_into(op, y, buf_a, buf_b, deg, window):
    """Run K1 deg times; y is read (may be buf_b for in-place). Returns the
    buffer holding the result."""
    res = ctypes.c_void_p()
    n, w = y.shape
    check(lib().chfsi_filter_z(ctx(), n, w, dptr(op.tensor), op.ld, op.conj, dptr(y), ld_of(y),
                               dptr(buf_a), dptr(buf_b), ld_of(buf_a), deg, float(window.a),
                               float(window.b), float(window.scale_ref), ctypes.byref(res)),
          "chebyshev_filter")
    return buf_a if res.value == buf_a.data_ptr() else buf_b


def chebyshev_filter(h, y, deg, window):
    """Degree-``deg`` scaled Chebyshev filter of the block ``y``
    (chfsi.py:179-208) on the device; returns a new column-major device
    block, ``y`` is untouched. ``deg`` may also be a sequence of per-column
    degrees (additive): column j is then filtered with degree
    ``deg[j]``."""
    host = host_output(h, y)
    op = Operator.wrap(h)
    ym = to_fblock(y)
    if ym.shape[0] != op.n:
        raise ValueError(f"operator/block shapes do not conform: {(op.n, op.n)} vs {tuple(ym.shape)}")
    n, w = ym.shape
    if np.ndim(deg) == 0:
        if deg < 1:
            raise ValueError("polynomial degree must be >= 1")
        a, b = fblock(n, w), fblock(n, w)
        return emit(_filter_into(op, ym, a, b, int(deg), window), host)
    degs = np.asarray(deg, dtype=np.int64)
    if degs.shape != (w,) or (degs < 1).any():
        raise ValueError("need one polynomial degree >= 1 per column")
    order = np.argsort(degs, kind="stable")
    ident = bool((order == np.arange(w)).all())
    ys = ym if ident else ym.index_select(1, torch.from_numpy(order).to(ym.device))
    ys = to_fblock(ys)
    a, b = fblock(n, w), fblock(n, w)
    sd = np.ascontiguousarray(degs[order], dtype=np.int32)
    res = ctypes.c_void_p()
    check(lib().chfsi_filter_degrees_z(ctx(), n, w, dptr(op.tensor), op.ld, op.conj, dptr(ys),
                                       ld_of(ys), dptr(a), dptr(b), ld_of(a),
                                       sd.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                       float(window.a), float(window.b), float(window.scale_ref),
                                       ctypes.byref(res)), "chebyshev_filter")
    out = a if res.value == a.data_ptr() else b
    if ident:
        return emit(out, host)
    inv = np.empty(w, dtype=np.int64)
    inv[order] = np.arange(w)
    return emit(to_fblock(out.index_select(1, torch.from_numpy(inv).to(out.device))), host)


def chebyshev_response(lam, deg, window):
    """Scalar filter response s_deg(lam) (chfsi.py:211-225) — host numpy:
    it is the filter's own oracle, evaluated on eigenvalues only."""
    lam = np.asarray(lam, dtype=float)
    e = (window.b - window.a) / 2
    c = (window.b + window.a) / 2
    sigma = e / (window.scale_ref - c)
    tau = 2.0 / sigma
    s_prev = np.ones_like(lam)
    s_cur = (sigma / e) * (lam - c)
    for _ in range(deg - 1):
        sigma_new = 1.0 / (tau - sigma)
        s_next = (2 * sigma_new / e) * (lam - c) * s_cur - (sigma * sigma_new) * s_prev
        s_prev, s_cur, sigma = s_cur, s_next, sigma_new
    return s_cur


# ---------------------------------------------------------- Rayleigh-Ritz ---

def _apply_h(op, y, out):
    check(lib().chfsi_cheb_step_z(ctx(), op.n, y.shape[1], dptr(op.tensor), op.ld, op.conj,
                                  dptr(y), ld_of(y), None, 0, dptr(out), ld_of(out), 1.0, 0.0,
                                  0.0), "H @ panel")


def _gemm(ta, tb, m, n, k, a, b, c, alpha=1.0, beta=0.0):
    check(lib().chfsi_gemm_z(ctx(), ta, tb, m, n, k, alpha, 0.0, dptr(a), ld_of(a), dptr(b),
                             ld_of(b), beta, 0.0, dptr(c), ld_of(c)), "zgemm")


# Off-diagonal target of the near-diagonal Rayleigh-Ritz eigensolver, relative
# to max|G_ii|: its remainder enters the Ritz residuals directly, so it must sit
# far below the locking tolerance (1e-13 * ||G|| vs tol = 1e-10 at BASELINE).
RR_FAST_TOL = 1e-13


def _rr_core(op, panel, hp, g, rot_p, rot_hp, ritz_d, res_d, eig_tol=0.0):
    """HP = H P; G = P^H HP, symmetrized; eigendecomposition; P W, HP W;
    residual norms (chfsi.py:341-350). All device. With ``eig_tol > 0`` the
    near-diagonal Jacobi/ZGEMM eigensolver is tried before zheevd. Returns
    True when it was used."""
    n, w = panel.shape
    _apply_h(op, panel, hp)
    _gemm(b"C", b"N", w, w, n, panel, hp, g)
    check(lib().chfsi_symmetrize_z(ctx(), w, dptr(g), ld_of(g)), "symmetrize")
    used = ctypes.c_int(0)
    check(lib().chfsi_heev_rr_z(ctx(), w, dptr(g), ld_of(g), dptr(ritz_d), float(eig_tol),
                                ctypes.byref(used)), "hermitian_eig")
    _gemm(b"N", b"N", n, w, w, panel, g, rot_p)
    _gemm(b"N", b"N", n, w, w, hp, g, rot_hp)
    check(lib().chfsi_colnorm_residual_z(ctx(), n, w, dptr(rot_hp), ld_of(rot_hp), dptr(rot_p),
                                         ld_of(rot_p), dptr(ritz_d), dptr(res_d)), "residuals")
    return bool(used.value)


def rayleigh_ritz(h, y):
    """Rayleigh-Ritz projection onto the orthonormal block ``y``
    (chfsi.py:228-239): ascending Ritz values (host) and ``y @ w``."""
    host = host_output(h, y)
    op = Operator.wrap(h)
    ym = to_fblock(y)
    n, w = ym.shape
    hp, rot_p, rot_hp = fblock(n, w), fblock(n, w), fblock(n, w)
    g = fblock(w, w)
    ritz_d = torch.empty(w, dtype=torch.float64, device=ym.device)
    res_d = torch.empty(w, dtype=torch.float64, device=ym.device)
    _rr_core(op, ym, hp, g, rot_p, rot_hp, ritz_d, res_d)
    return ritz_d.cpu().numpy(), emit(rot_p, host)


# ------------------------------------------------------------ orthonormal ---

class _LoopCallbacks:
    """Host callbacks of the native loop: rank-repair draws from the
    caller's Generator (reference order, chfsi.py:255-259) and, in the
    row-sharded multi-GPU loop, the sharded filter, H*P, the all-reduce of
    partial Grams / norms and the gather for the full-matrix fallbacks.
    Exceptions raised in a callback are re-raised after the loop returns."""

    def __init__(self, bufs, rows, rng, comm=None, op=None, blk=0, reduce_bufs=(), hp_buf=None):
        self.bufs, self.rows, self.rng = bufs, rows, rng
        self.hp_buf = hp_buf
        self.comm, self.op, self.blk = comm, op, blk
        self.reduce_bufs = list(reduce_bufs)  # device tensors the loop all-reduces
        self.full = None                      # scratch of the gather fallback
        self.error = None
        self.fill_cb = FILL_CB(self._fill)
        if comm is not None:  # (ctypes thunks cost ~10 us each: only the sharded loop needs these)
            self.filter_cb = FILTER_CB(self._filter)
            self.allreduce_cb = ALLREDUCE_CB(self._allreduce)
            self.hp_cb = HP_CB(self._hp)
            self.gather_cb = GATHER_CB(self._gather)

    def _view(self, ptr, width):
        for b in self.bufs:
            off = (ptr - b.data_ptr()) // (16 * self.rows)
            if 0 <= off < b.shape[1] and b.data_ptr() + off * 16 * self.rows == ptr:
                return b[:, off:off + width]
        raise ValueError("pointer outside the panel buffers")

    def _guard(self, fn, *args):
        try:
            fn(*args)
            return 0
        except BaseException as exc:  # noqa: BLE001 - re-raised by reraise()
            self.error = exc
            return -1

    def _fill(self, user, block, ld, rows, cols, ncols):
        def run():
            idx = [cols[j] for j in range(ncols)]
            work = self._view(block, max(idx) + 1)
            n = self.comm.part.n if self.comm is not None else self.rows
            fresh = random_block(self.rng, n, ncols)  # every rank draws the full columns
            if self.comm is not None:
                fresh = fresh[self.comm.part.r0:self.comm.part.r0 + self.rows]
            for j, c in enumerate(idx):
                work[:, c].copy_(fresh[:, j])

        return self._guard(run)

    def _filter(self, user, panel, other, ld, width, deg, degs, a, b, scale_ref, result):
        def run():
            d = [degs[j] for j in range(width)] if degs else deg
            win = FilterWindow(a=a, b=b, scale_ref=scale_ref)
            out = self.comm.filter_local(self.op, self.blk, self._view(panel, width), d, win,
                                         self._view(other, width))
            result[0] = out.data_ptr()

        return self._guard(run)

    def _allreduce(self, user, buf, count):
        def run():
            for t in self.reduce_bufs:
                base = t.t() if (t.dim() == 2 and t.stride(0) == 1) else t  # F-block storage
                flat = (torch.view_as_real(base) if base.is_complex() else base).view(-1)
                off = (buf - base.data_ptr()) // 8
                if 0 <= off and off + count <= flat.numel() and base.data_ptr() + 8 * off == buf:
                    self.comm.allreduce_(flat[off:off + count])
                    return
            raise ValueError("allreduce pointer outside the reduction buffers")

        return self._guard(run)

    def _hp(self, user, panel, out, ld, width):
        def run():
            assert out == self.hp_buf.data_ptr()
            self.comm.hp_local(self.op, self._view(panel, width), self.hp_buf[:, :width])

        return self._guard(run)

    def _gather(self, user, local, ld, width, full_out):
        def run():
            n = self.comm.part.n
            if self.full is None or self.full.shape[1] < width:
                self.full = fblock(n, max(width, self.blk), self.bufs[0].device)
            full = self.full[:, :width]
            self.comm.gather_rows(self._view(local, width), full)
            full_out[0] = full.data_ptr()

        return self._guard(run)

    def reraise(self):
        if self.error is not None:
            err, self.error = self.error, None
            raise err


_WORKSPACES = {}


def _workspace(dev, n, blk, nev):
    """HBM workspace of one solve, reused by the next solve of the same shape
    on the same stream (a sequence allocates it once): two panel buffers
    (filter ping-pong / rotation target), two H*panel buffers, the locked
    block, the projected matrix, CGS coefficients, Ritz values, residuals.
    Nothing returned to the caller aliases it."""
    key = (dev, torch.cuda.current_stream(dev).cuda_stream, n, blk, nev)
    ws = _WORKSPACES.get(key)
    if ws is None:
        if len(_WORKSPACES) >= 4:  # bound the cache: drop the oldest shape
            _WORKSPACES.pop(next(iter(_WORKSPACES)))
        # (Ritz values | residuals) as the halves of one buffer: the native
        # loop then reads both back in one copy per pass
        rr = torch.empty(2 * blk, dtype=torch.float64, device=dev)
        ws = _WORKSPACES[key] = (
            [fblock(n, blk, dev), fblock(n, blk, dev)], fblock(n, blk, dev), fblock(n, blk, dev),
            fblock(n, max(nev, 1), dev), fblock(blk, blk, dev), fblock(max(nev, 1), blk, dev),
            rr[:blk], rr[blk:],
            torch.empty(blk, dtype=torch.int32, device=dev))
    return ws


def _safe_window(scale_ref, a, b):
    """Clamp a refreshed window back to scale_ref < a < b (chfsi.py:264-271)."""
    if not np.isfinite([scale_ref, a, b]).all() or not scale_ref < b:
        return FilterWindow(a=scale_ref + 0.5, b=scale_ref + 1.0, scale_ref=scale_ref)
    if not scale_ref < a < b:
        a = scale_ref + 0.5 * (b - scale_ref)
    return FilterWindow(a=a, b=b, scale_ref=scale_ref)


# ----------------------------------------------------------------- solver ---

@dataclass
class WarmLanczos:
    """A warm start's Lanczos bound estimate computed ahead of the solve
    (`warm_lanczos`): the generator (already past the q0 draw, so later
    draws continue the reference's stream) and the estimate."""
    rng: np.random.Generator
    ritz: np.ndarray
    beta_last: float
    steps: int


def warm_lanczos(h, seed):
    """The spectral-bound estimate of a warm start (chfsi.py:301-305 as called
    from chfsi.py:309-316: ten Lanczos steps from a fresh q0) on torch's
    current stream, ahead of the solve. Returns None on any failure (the
    solve then computes it itself, after the pencil's validation)."""
    try:
        rng = np.random.default_rng(seed)
        op = Operator.wrap(h)
        ritz, beta_last, steps = _lanczos_estimates(op, min(10, op.n), rng)
        if not (np.isfinite(ritz).all() and np.isfinite(beta_last)):
            return None
        return WarmLanczos(rng=rng, ritz=ritz, beta_last=float(beta_last), steps=int(steps))
    except Exception:  # noqa: BLE001  (e.g. a pencil that fails validation: reported by the solve path)
        return None


def chfsi_solve(h, cfg, guess=None, rng=None, label=1, *, shard=None, _hooks=None, _sync=True,
                _out=None, _warm=None):
    """Compute the ``cfg.nev`` lowest eigenpairs of the Hermitian ``h``
    (chfsi.py:274-384). ``h`` may be a numpy array (uploaded once) or a CUDA
    tensor in either row- or column-major layout (used in place).

    ``shard`` (multi-GPU): ``True``, a torch.distributed process
    group or a `distributed.RowComm` runs the row-sharded loop: every rank
    (one GPU each, all calling chfsi_solve with the same arguments) keeps its
    rows of every n x w block, the filter and H*P run as row-sharded K1
    steps (fused all-gather over NVLink with NCCL), and the w x w Grams and
    residual norms are all-reduced; Lanczos and the w x w eigenproblems are
    replicated from identical inputs. ``shard=k`` (int) also sets the number
    of column groups of the unfused filter. Every rank returns the same full
    solution; ``report.tail_vectors`` holds this rank's rows.

    Returns ``(EigenSolution(form="standard"), SolveReport)``. The solution
    vectors are numpy when ``h`` (and the guess) came from host memory, as
    in the reference, and stay on the device for device inputs
    (`set_array_output`); ``report.tail_vectors`` always stays on the device.
    """
    t0 = time.perf_counter()
    host = host_output(h, None if guess is None else guess.vectors)
    pre = rng if isinstance(rng, PrefetchedStart) else None
    rng = pre.rng if pre is not None else as_rng(rng)
    op = Operator.wrap(h)
    n = op.n
    blk, deg, tol, lancz_k, max_repeats = cfg.resolve(n)
    if pre is not None and (guess is not None or (pre.n, pre.blk) != (n, blk)):
        raise ValueError("prefetched cold-start draws need a cold start of the same n and blk")
    report = SolveReport()
    dev = op.tensor.device
    t_lz = _PhaseTimer()
    comm = None
    if shard is not None and shard is not False:
        from .distributed import RowComm

        if hasattr(shard, "part") and hasattr(shard, "allreduce_"):
            comm = shard  # a RowComm (or a stand-in with the same interface)
        else:
            group = shard if not isinstance(shard, (bool, int)) else None
            chunks = shard if isinstance(shard, int) and not isinstance(shard, bool) else 2
            comm = RowComm(n, group=group, chunks=chunks)
    r0, rows = (comm.part.r0, comm.part.rows) if comm is not None else (0, n)
    if rows < 1:
        raise ValueError("every rank needs at least one row of the problem")

    bufs, hp_buf, hp_rot, locked, g_buf, coef, ritz_d, res_d, perm_d = _workspace(dev, rows, blk,
                                                                                 cfg.nev)

    hw = {"setup": time.perf_counter() - t0}
    t_lz.start()
    if guess is not None:
        gv = guess.vectors
        shape = tuple(gv.shape)
        if shape not in ((n, blk), (rows, blk)):
            raise ValueError(f"guess block must be {n}x{blk}, got {shape}")
        if _warm is not None and comm is None:  # estimated ahead (sequence driver), same rng stream
            ritz, beta_last, steps = _warm.ritz, _warm.beta_last, _warm.steps
        else:
            ritz, beta_last, steps = _lanczos_estimates(op, min(10, n), rng, comm=comm)
        b_up = float(ritz[-1] + beta_last)
        window = _safe_window(guess.lambda1, guess.lambda_blk_plus_1, b_up)
        gv = to_fblock(gv)
        bufs[0].copy_(gv if gv.shape[0] == rows else gv[r0:r0 + rows])
    else:
        # The start block is the next draw after the Lanczos vector
        # (chfsi.py:137 then chfsi.py:323): draw q0, then let a host thread
        # draw the block (numpy releases the GIL) while the device runs the
        # Lanczos chain — same stream of numbers, ~10 ms less at C2.
        if pre is None:  # draw here (the block on a host thread, staged page-locked)
            pre = PrefetchedStart(rng, n, blk)
        q0 = pre.q0()
        try:
            ritz, beta_last, steps = _lanczos_estimates(op, lancz_k, rng, q0=q0, comm=comm)
        finally:
            zblock = pre.block()
        b_up = float(ritz[-1] + beta_last)
        if ritz.size > blk:
            a = float(ritz[blk])
        else:
            a = float(ritz[-1] - 0.10 * (ritz[-1] - ritz[0]))
        window = _safe_window(float(ritz[0]), a, b_up)
        start = to_fblock(zblock)
        qr_orthonormalize_inplace(start)  # full block on every rank (replicated)
        bufs[0].copy_(start if rows == n else start[r0:r0 + rows])
    t_lz.stop()
    report.lanczos_matvecs = steps
    report.matvecs += steps
    report.operator_norm_estimate = float(max(abs(ritz[0]), abs(ritz[-1])) + beta_last)

    # ---- the inner loop runs natively (chfsi_solve_loop_z, chfsi_loop.cu)
    st = LoopState()
    st.n, st.blk, st.nev, st.deg, st.max_repeats = n, blk, cfg.nev, deg, max_repeats
    st.tol = tol
    # near-diagonal Rayleigh-Ritz eigensolver first (bails out to zheevd when
    # the projection is not close to diagonal)
    st.rr_fast_tol = RR_FAST_TOL if tol >= 1e-11 else 0.0
    st.reuse_hp = 0 if os.environ.get("CHFSI_REUSE_HP") == "0" else 1
    st.H, st.ldh, st.conj_h = op.tensor.data_ptr(), op.ld, int(op.conj)
    st.bufs[0], st.bufs[1] = bufs[0].data_ptr(), bufs[1].data_ptr()
    st.hp, st.hp_rot, st.locked = hp_buf.data_ptr(), hp_rot.data_ptr(), locked.data_ptr()
    st.g, st.coef = g_buf.data_ptr(), coef.data_ptr()
    st.ritz_d, st.res_d, st.perm_d = ritz_d.data_ptr(), res_d.data_ptr(), perm_d.data_ptr()
    st.adaptive, st.deg_min = int(cfg.adaptive_degree), int(cfg.min_degree)
    # (_out: the sequence driver's preallocated (tail, vectors) blocks)
    tail = _out[0] if _out is not None else fblock(rows, blk, dev)
    st.tail = tail.data_ptr()
    st.win_a, st.win_b, st.win_scale_ref = window.a, window.b, window.scale_ref
    st.pb, st.off, st.width = 0, 0, blk
    host_f = np.zeros((4, blk))
    locked_per_loop = np.zeros(max(max_repeats, 1), dtype=np.int32)
    pd_, pi_ = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
    st.locked_vals = host_f[0].ctypes.data_as(pd_)
    st.locked_res = host_f[1].ctypes.data_as(pd_)
    st.ritz = host_f[2].ctypes.data_as(pd_)
    st.res = host_f[3].ctypes.data_as(pd_)
    host_degs = np.zeros(blk, dtype=np.int32)
    st.degs = host_degs.ctypes.data_as(pi_)
    st.locked_per_loop = locked_per_loop.ctypes.data_as(pi_)
    callbacks = _LoopCallbacks(bufs, rows, rng, comm, op, blk, reduce_bufs=(coef, g_buf, res_d),
                               hp_buf=hp_buf)
    st.fill = callbacks.fill_cb
    if comm is not None:  # row-sharded loop: local rows + collectives
        st.row0, st.n_local = r0, rows
        st.filter = callbacks.filter_cb
        st.allreduce = callbacks.allreduce_cb
        st.hp_fn = callbacks.hp_cb
        st.gather = callbacks.gather_cb
    hw["lanczos_start"] = time.perf_counter() - t0 - hw["setup"]
    if _hooks is not None:  # (sequence driver: hand queued side-stream work to its worker)
        _hooks()
    t_loop = time.perf_counter()
    status = lib().chfsi_solve_loop_z(ctx(), ctypes.byref(st))
    hw["loop"] = time.perf_counter() - t_loop
    callbacks.reraise()
    check(status, "chfsi inner loop")

    nlocked = st.nlocked
    report.inner_loops = st.inner_loops
    report.filtered_vectors = int(st.filtered_vectors)
    report.matvecs += int(st.matvecs)
    report.residual_check_matvecs = int(st.residual_check_matvecs)
    report.filter_launches = int(st.filter_launches)
    report.filter_flops = float(st.filter_flops)
    report.filter_k1_launches = int(st.filter_k1_launches)
    report.filter_k1_flops = float(st.filter_k1_flops)
    report.filter_degree_sum = int(st.filter_degree_sum)
    report.rr_fast_eigs = int(st.rr_fast_eigs)
    report.qr_redone = int(st.qr_redone)
    report.converged = bool(st.converged)
    report.locked_per_loop = [int(x) for x in locked_per_loop[: st.inner_loops]]
    locked_vals = host_f[0, :nlocked].tolist()
    locked_res = host_f[1, :nlocked].tolist()

    # chained-mode tail [locked | unlocked remainder of the final panel],
    # assembled by the native loop (always exactly blk columns)
    if st.inner_loops:
        report.tail_vectors = tail
        report.lambda_blk_plus_1 = float(host_f[2, st.last_width - 1])

    order = np.argsort(locked_vals, kind="stable")
    vecs = locked[:, :nlocked]
    if nlocked and not np.array_equal(order, np.arange(nlocked)):
        idx = torch.from_numpy(order).to(dev)
        vecs = vecs.index_select(1, idx)
    if comm is not None:  # every rank returns the full vectors
        full = fblock(n, nlocked, dev)
        vecs = comm.gather_rows(to_fblock(vecs, copy=True), full)
    if host:
        vecs = to_host(vecs)
    elif _out is not None and not nlocked:
        vecs = _out[1][:, :0]
    elif _out is not None:
        dst = _out[1][:, :nlocked]
        dst.copy_(vecs)
        vecs = dst
    else:
        vecs = to_fblock(vecs, copy=True)
    sol = EigenSolution(values=np.asarray(locked_vals)[order], vectors=vecs, form="standard",
                        label=label)
    report.final_residuals = np.asarray(locked_res)[order]
    if _sync:
        torch.cuda.current_stream().synchronize()
    report.t_lanczos = t_lz.seconds()
    report.t_filter = st.t_filter
    report.t_ortho = st.t_ortho
    report.t_rr = st.t_rr
    report.wall_time = time.perf_counter() - t0
    hw["finish"] = report.wall_time - sum(hw.values())
    report.host_phases = hw
    return sol, report
