"""Binary pencil/sequence persistence.

Replaces the reference's Matrix Market text files (`pencil_io.py:30-121`,
17-digit text: ~8 GB and minutes per n=20000 matrix) with raw complex128
`.npy` files: a sequence directory holds ``A_<l>.npy`` / ``B_<l>.npy`` per
problem plus a ``manifest.json`` with the same keys as the reference's
(``n``, ``length``, ``provenance``) and ``"format": "npy"``. Files are read
memory-mapped, so a C5 sequence (76 GB) streams one pencil at a time, and
bytes round-trip exactly. Reference-format directories (``*.mtx``) are
still readable (scipy), so an existing data set switches over unchanged.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

__all__ = ["FormatError", "write_pencil", "read_pencil", "save_sequence", "load_sequence",
           "iter_sequence"]


class FormatError(ValueError):
    """Pencil file is malformed or declares an unsupported format
    (same class name and meaning as the reference, pencil_io.py:33-34)."""


def _npy(directory, name, label):
    return Path(directory) / f"{name}_{label}.npy"


def _mtx(directory, name, label):
    return Path(directory) / f"{name}_{label}.mtx"


def _as_host(m):
    try:
        import torch

        if isinstance(m, torch.Tensor):
            return m.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(m)


def _read_matrix(directory, name, label, mmap=True):
    p = _npy(directory, name, label)
    if p.is_file():
        try:
            m = np.load(p, mmap_mode="r" if mmap else None, allow_pickle=False)
        except Exception as exc:  # noqa: BLE001
            raise FormatError(f"{p}: unreadable npy ({exc})") from exc
        if m.ndim != 2 or m.shape[0] != m.shape[1] or m.dtype != np.complex128:
            raise FormatError(f"{p}: expected a square complex128 matrix, got {m.shape} {m.dtype}")
        return m
    q = _mtx(directory, name, label)
    if q.is_file():  # reference Matrix Market format
        import scipy.io

        try:
            return np.asarray(scipy.io.mmread(str(q)), dtype=np.complex128)
        except Exception as exc:  # noqa: BLE001
            raise FormatError(f"malformed Matrix Market file {q}: {exc}") from exc
    raise FormatError(f"missing matrix file {p}")


def write_pencil(pencil, directory, label=None):
    """Write one pencil (EigenPencil or (label, A, B)) as A_<l>.npy / B_<l>.npy."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    if isinstance(pencil, tuple):
        lab, a, b = pencil
    else:
        lab, a, b = pencil.label, pencil.a, pencil.b
    lab = lab if label is None else label
    a, b = _as_host(a), _as_host(b)
    if a.shape != b.shape or a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise FormatError(f"pencil {lab}: A and B must be square and conform")
    np.save(_npy(directory, "A", lab), np.ascontiguousarray(a, dtype=np.complex128))
    np.save(_npy(directory, "B", lab), np.ascontiguousarray(b, dtype=np.complex128))
    return lab


def read_pencil(directory, label=1, device=False):
    """Read pencil ``label``: ``(label, A, B)`` host arrays (memory-mapped),
    or a device EigenPencil (validated Hermitian) with ``device=True``."""
    a = _read_matrix(directory, "A", label)
    b = _read_matrix(directory, "B", label)
    if a.shape != b.shape:
        raise FormatError(f"A_{label} and B_{label} differ in dimension: {a.shape} vs {b.shape}")
    if not device:
        return label, a, b
    from .linalg_errors import NotHermitianError
    from .reduction import EigenPencil

    try:
        return EigenPencil(a=np.ascontiguousarray(a), b=np.ascontiguousarray(b), label=label)
    except (NotHermitianError, ValueError) as exc:
        raise FormatError(f"pencil {label} rejected: {exc}") from exc


def save_sequence(pencils, directory, provenance=None):
    """Write every pencil of an iterable (streamed) plus the manifest."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    n, length = None, 0
    for expected, p in enumerate(pencils, start=1):
        lab = write_pencil(p, directory)
        if lab != expected:
            raise FormatError(f"labels must run 1..N, found {lab} at position {expected}")
        a = p[1] if isinstance(p, tuple) else p.a
        n = a.shape[0] if n is None else n
        if a.shape[0] != n:
            raise FormatError("all pencils must share one dimension")
        length = expected
    manifest = {"n": n, "length": length, "format": "npy", "provenance": provenance or {}}
    with open(directory / "manifest.json", "w") as fh:
        json.dump(manifest, fh, indent=2)
    return manifest


def _manifest(directory):
    path = Path(directory) / "manifest.json"
    if not path.is_file():
        raise FormatError(f"missing manifest.json in {directory}")
    try:
        with open(path) as fh:
            m = json.load(fh)
        return int(m["n"]), int(m["length"]), m
    except (json.JSONDecodeError, KeyError, TypeError, ValueError) as exc:
        raise FormatError(f"malformed manifest in {directory}: {exc}") from exc


def iter_sequence(directory):
    """Lazily yield ``(label, A, B)`` (memory-mapped) for labels 1..N."""
    n, length, _ = _manifest(directory)
    for label in range(1, length + 1):
        lab, a, b = read_pencil(directory, label)
        if a.shape[0] != n:
            raise FormatError(f"pencil {label} has dimension {a.shape[0]}, manifest says {n}")
        yield lab, a, b


def load_sequence(directory):
    """All ``(label, A, B)`` of a directory (memory-mapped npy, or the
    reference's Matrix Market files) — feeds `solve_sequence` directly."""
    return list(iter_sequence(directory))
