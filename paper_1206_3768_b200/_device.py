"""Device-memory plumbing: complex128 blocks in HBM as torch tensors.

Layout rules of the device path:
* n x w blocks (panels, locked vectors, H*panel, eigenvectors) are
  column-major "F-blocks": a torch tensor of shape (n, w) with strides
  (1, ld), ld >= n — each column contiguous, so column slices and locking
  are pointer offsets and cuBLAS/cuSOLVER use them without transposes.
* The operator H of K1/K2 may be row-major (as numpy hands it over) or
  column-major (as the device reduction produces it); Hermitian symmetry
  makes the second the conjugate of the first, so the kernels just flip a
  `conj` flag instead of transposing 16 n^2 bytes.
"""

from __future__ import annotations

import contextlib
import os
import threading

import numpy as np
import torch

from ._lib import BackendUnavailable

C128 = torch.complex128


def device():
    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device visible: the ChFSI path runs only on the GPU")
    return torch.device("cuda", torch.cuda.current_device())


def fblock(n, w, dev=None):
    """Uninitialised column-major n x w complex128 block on the device."""
    return torch.empty((w, n), dtype=C128, device=dev or device()).t()


def is_fblock(t):
    return (
        isinstance(t, torch.Tensor)
        and t.is_cuda
        and t.dtype == C128
        and t.dim() == 2
        and (t.stride(0) == 1 or t.shape[0] <= 1)
        and (t.shape[1] <= 1 or t.stride(1) >= t.shape[0])
    )


def ld_of(t):
    """Leading dimension of an F-block (>= rows, as BLAS requires)."""
    return max(int(t.stride(1)) if t.shape[1] > 1 else int(t.shape[0]), int(t.shape[0]), 1)


def _as_tensor(x):
    if isinstance(x, torch.Tensor):
        return x
    a = np.asarray(x)
    if a.ndim == 1:
        a = a[:, None]
    if a.dtype != np.complex128:
        a = a.astype(np.complex128)
    return torch.from_numpy(a)


def to_fblock(x, copy=False):
    """Device F-block view of ``x`` (numpy or torch, any strides).

    Zero-copy when ``x`` already is a device complex128 F-block and
    ``copy`` is False; otherwise one H2D/D2D copy into a fresh block.
    """
    if not copy and is_fblock(x):
        return x
    t = _as_tensor(x)
    if t.dim() == 1:
        t = t[:, None]
    if t.dim() != 2:
        raise ValueError(f"expected a 2-D block, got shape {tuple(t.shape)}")
    out = fblock(t.shape[0], t.shape[1])
    if t.dtype != C128:
        t = t.to(C128)
    out.copy_(t, non_blocking=True)
    return out


def to_device_matrix(x):
    """Device complex128 square matrix, keeping row-major input row-major."""
    t = _as_tensor(x)
    if t.dim() != 2:
        raise ValueError(f"expected a matrix, got shape {tuple(t.shape)}")
    if t.dtype != C128:
        t = t.to(C128)
    dev = device()
    if t.device != dev:
        t = t.to(dev, non_blocking=True)
    return t


class Operator:
    """The Hermitian operator H as the kernels read it (pointer, ld, conj).
    ``row0``: global index of the first row the storage holds (0 for a full
    H; `distributed.RowOperator` holds one rank's row block)."""

    __slots__ = ("tensor", "n", "ld", "conj", "row0", "rows")

    def __init__(self, h):
        t = to_device_matrix(h)
        n = t.shape[0]
        if t.shape != (n, n):
            raise ValueError(f"operator must be square, got {tuple(t.shape)}")
        if n > 1 and t.stride(1) == 1 and t.stride(0) >= n:
            conj, ld = 0, t.stride(0)          # row-major H
        elif n > 1 and t.stride(0) == 1 and t.stride(1) >= n:
            conj, ld = 1, t.stride(1)          # column-major H == conj(H) row-major
        else:
            t = t.contiguous()
            conj, ld = 0, max(n, 1)
        self.tensor, self.n, self.ld, self.conj = t, n, ld, conj
        self.row0, self.rows = 0, n

    def row_ptr(self, r0, rows):
        """Device address of rows [r0, r0+rows) as K1 reads them (row-major
        stride ld; for column-major storage the conj flag makes column r
        read as row r)."""
        if r0 < self.row0 or r0 + rows > self.row0 + self.rows:
            raise ValueError(f"rows [{r0}, {r0 + rows}) are not held by this operator "
                             f"([{self.row0}, {self.row0 + self.rows}))")
        return self.tensor.data_ptr() + (r0 - self.row0) * self.ld * 16

    @classmethod
    def wrap(cls, h):
        return h if isinstance(h, Operator) else cls(h)


def to_host(x):
    """numpy copy of a device tensor (test/report helper)."""
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


# ------------------------------------------------------ array payloads ---
# The reference returns numpy arrays (linalg.py:5-6: "outputs are fresh
# arrays") and its callers do numpy arithmetic on them (harness.py:263-265,
# sequence.py:209). Policy for the n-sized outputs of the drop-in functions:
#   "auto"  (default) numpy out when every array input was host memory
#           (numpy / lists), CUDA tensors out when any input was a CUDA
#           tensor — a numpy caller gets the reference's types, a device
#           caller keeps everything in HBM;
#   "numpy" always numpy;   "torch" always device tensors.
# The arithmetic runs on the device either way; "numpy" only adds the D2H.
_OUTPUT_MODES = ("auto", "numpy", "torch")
_output_default = os.environ.get("CHFSI_ARRAY_OUTPUT", "auto")
if _output_default not in _OUTPUT_MODES:
    raise ValueError(f"CHFSI_ARRAY_OUTPUT must be one of {_OUTPUT_MODES}, got {_output_default!r}")
_output_local = threading.local()


def set_array_output(mode):
    """Set the process-wide payload policy ("auto", "numpy" or "torch")."""
    global _output_default
    if mode not in _OUTPUT_MODES:
        raise ValueError(f"array output mode must be one of {_OUTPUT_MODES}, got {mode!r}")
    _output_default = mode


def get_array_output():
    return getattr(_output_local, "mode", None) or _output_default


@contextlib.contextmanager
def array_output(mode):
    """Thread-local override of the payload policy inside a with-block."""
    if mode not in _OUTPUT_MODES:
        raise ValueError(f"array output mode must be one of {_OUTPUT_MODES}, got {mode!r}")
    prev = getattr(_output_local, "mode", None)
    _output_local.mode = mode
    try:
        yield
    finally:
        _output_local.mode = prev


def host_output(*inputs):
    """True when the outputs of a call on ``inputs`` go back as numpy."""
    mode = get_array_output()
    if mode != "auto":
        return mode == "numpy"
    return not any(isinstance(x, (torch.Tensor, Operator)) or getattr(x, "device_input", False)
                   for x in inputs if x is not None)


def emit(x, host):
    """``x`` as the caller's payload type (numpy copy when ``host``)."""
    return to_host(x) if host and isinstance(x, torch.Tensor) else x
