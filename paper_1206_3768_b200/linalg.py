"""Dense complex kernels on the device — drop-in for `spectral_chain.linalg`.

Same names, argument meaning and exceptions as the reference
(`spectral_chain/linalg.py`), computed in HBM by libchfsi (hand-written
sm_100a kernels plus cuBLAS/cuSOLVER for the factorizations). Inputs may be
numpy arrays (uploaded) or CUDA tensors (used in place); outputs are numpy
arrays for host inputs (as the reference's) and CUDA tensors in column-major
"F-block" layout for device inputs (`_device.py`, `set_array_output`).
Inputs are never modified.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._device import Operator, emit, fblock, host_output, ld_of, to_device_matrix, to_fblock
from ._lib import check, ctx, dptr, lib
from .linalg_errors import (
    EigenSolverError,
    NotHermitianError,
    NotPositiveDefiniteError,
    RankDeficientError,
)

__all__ = [
    "NotHermitianError",
    "NotPositiveDefiniteError",
    "RankDeficientError",
    "EigenSolverError",
    "hermitian_view",
    "gemm",
    "cholesky",
    "triangular_solve",
    "qr_orthonormalize",
    "hermitian_eig",
]


def hermitian_defect(m):
    """(max|m - m^H|, max|m|) of a device square matrix (linalg.py:78-81)."""
    t = to_device_matrix(m)
    n = t.shape[0]
    if n == 0:
        return 0.0, 0.0
    op = Operator(t)  # any layout: the defect of A^T equals that of A
    d = ctypes.c_double()
    a = ctypes.c_double()
    check(lib().chfsi_herm_defect_z(ctx(), n, dptr(op.tensor), op.ld, ctypes.byref(d),
                                    ctypes.byref(a)), "hermitian_defect")
    return d.value, a.value


def hermitian_view(m, tol=None):
    """Validate that ``m`` is Hermitian (linalg.py:61-85); returns it as a
    complex128 array of the caller's payload type. Raises NotHermitianError."""
    host = host_output(m)
    t = _hermitian_device(m, tol)
    return np.asarray(m, dtype=np.complex128) if host and not isinstance(m, torch.Tensor) \
        else emit(t, host)


def _hermitian_device(m, tol=None):
    """hermitian_view's check, returning the device tensor (internal)."""
    t = to_device_matrix(m)
    if t.dim() != 2 or t.shape[0] != t.shape[1]:
        raise NotHermitianError(f"expected a square matrix, got shape {tuple(t.shape)}")
    defect, scale = hermitian_defect(t)
    if tol is None:
        tol = 1e-10 * max(1.0, scale)
    if defect > tol:
        raise NotHermitianError(f"symmetry defect {defect:.3e} exceeds tolerance {tol:.3e}")
    return t


_OPS = ("N", "T", "C")


def gemm(alpha, a, b, beta=0.0, c=None, trans_a="N", trans_b="N"):
    """``alpha * op(a) @ op(b) + beta * c`` on the device (linalg.py:91-113)."""
    if trans_a not in _OPS or trans_b not in _OPS:
        raise ValueError(f"unknown transpose flags ({trans_a!r}, {trans_b!r})")
    host = host_output(a, b, c)
    am, bm = to_fblock(a), to_fblock(b)
    m, ka = (am.shape[1], am.shape[0]) if trans_a != "N" else (am.shape[0], am.shape[1])
    kb, n = (bm.shape[1], bm.shape[0]) if trans_b != "N" else (bm.shape[0], bm.shape[1])
    if ka != kb:
        raise ValueError(f"inner dimensions do not conform: ({m}, {ka}) x ({kb}, {n})")
    if beta != 0.0:
        if c is None:
            raise ValueError("beta is nonzero but no c matrix was given")
        out = to_fblock(c, copy=True)
        if tuple(out.shape) != (m, n):
            raise ValueError(f"c has shape {tuple(out.shape)}, expected {(m, n)}")
    else:
        if c is not None and tuple(to_fblock(c).shape) != (m, n):
            raise ValueError("c does not conform to the product shape")
        out = fblock(m, n)
        out.zero_()
    al, be = complex(alpha), complex(beta)
    check(lib().chfsi_gemm_z(ctx(), trans_a.encode(), trans_b.encode(), m, n, ka, al.real, al.imag,
                             dptr(am), ld_of(am), dptr(bm), ld_of(bm), be.real, be.imag, dptr(out),
                             ld_of(out)), "gemm")
    return emit(out, host)


def cholesky(b):
    """Lower Cholesky factor with positive diagonal (linalg.py:116-129)."""
    host = host_output(b)
    t = _hermitian_device(b)
    n = t.shape[0]
    l = to_fblock(t, copy=True)
    info = ctypes.c_int()
    status = lib().chfsi_potrf_z(ctx(), n, dptr(l), ld_of(l), ctypes.byref(info))
    check(status, "cholesky")
    return emit(l, host)


def _diag_host(t):
    return torch.diagonal(t).cpu().numpy()


def triangular_solve(l, x, conjugate_transpose=False):
    """Solve ``L Z = X`` or ``L^H Z = X`` (linalg.py:132-149); never forms an inverse."""
    host = host_output(l, x)
    lm = to_fblock(l)
    xm = to_fblock(x, copy=True)
    if lm.shape[0] != lm.shape[1]:
        raise ValueError("triangular factor must be square")
    if lm.shape[0] != xm.shape[0]:
        raise ValueError(f"dimensions do not conform: {tuple(lm.shape)} vs {tuple(xm.shape)}")
    d = _diag_host(lm)
    if np.any(d.real <= 0.0) or np.any(d == 0.0):
        raise ValueError("triangular factor has a non-positive diagonal entry")
    check(lib().chfsi_trsm_z(ctx(), b"L", b"C" if conjugate_transpose else b"N", xm.shape[0],
                             xm.shape[1], dptr(lm), ld_of(lm), dptr(xm), ld_of(xm)),
          "triangular_solve")
    return emit(xm, host)


def qr_orthonormalize_inplace(y):
    """Q overwrites the packed device F-block ``y``; on rank deficiency ``y``
    is left untouched and RankDeficientError(indices) is raised."""
    m, n = y.shape
    if m < n:
        raise ValueError(f"need rows >= cols, got {(m, n)}")
    dead = (ctypes.c_int * max(n, 1))()
    nd = ctypes.c_int()
    status = lib().chfsi_qr_orthonormalize_z(ctx(), m, n, dptr(y), ld_of(y), dead, ctypes.byref(nd))
    if status == _lib.CHFSI_ERANK:
        raise RankDeficientError([dead[i] for i in range(nd.value)])
    check(status, "qr_orthonormalize")
    return y


def qr_orthonormalize(y):
    """Householder QR orthonormalization, positive-real R diagonal
    (linalg.py:152-178). Raises RankDeficientError when a column's
    post-projection norm falls below 1e-13 ||y||_F."""
    host = host_output(y)
    t = to_fblock(y, copy=True)
    if t.shape[0] < t.shape[1]:
        raise ValueError(f"need rows >= cols, got {tuple(t.shape)}")
    if ld_of(t) != t.shape[0]:
        t = t.contiguous().t().contiguous().t()
    return emit(qr_orthonormalize_inplace(t), host)


def hermitian_eig(g, want_vectors=True):
    """Full eigendecomposition of a Hermitian matrix (linalg.py:181-206).

    Returns ascending values (host numpy) and, when requested, the
    eigenvectors (device F-block, or numpy for a host input).
    """
    host = host_output(g)
    t = _hermitian_device(g)
    n = t.shape[0]
    a = to_fblock(t, copy=True)
    w = torch.empty(n, dtype=torch.float64, device=a.device)
    check(lib().chfsi_heevd_z(ctx(), n, dptr(a), ld_of(a), dptr(w)), "hermitian_eig")
    vals = w.cpu().numpy()
    return (vals, emit(a, host)) if want_vectors else (vals, None)
