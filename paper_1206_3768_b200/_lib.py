"""ctypes binding of libchfsi.so (the C-ABI declared in include/chfsi.h).

The product path has exactly one backend: this library on a CUDA device.
If the library is missing or no GPU is visible, every compute call raises
`BackendUnavailable` — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .linalg_errors import (
    EigenSolverError,
    NotPositiveDefiniteError,
    RankDeficientError,
)

__all__ = ["lib", "ctx", "BackendUnavailable", "check", "LIB_PATH", "symbols"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libchfsi.so")

CHFSI_OK = 0
CHFSI_EINVAL = -1
CHFSI_ECUDA = -2
CHFSI_ECUBLAS = -3
CHFSI_ECUSOLVER = -4
CHFSI_ENOTPD = -5
CHFSI_ERANK = -6
CHFSI_EEIG = -7
CHFSI_ENCCL = -8


class BackendUnavailable(RuntimeError):
    """libchfsi.so is not built or no CUDA device is available."""


class ChfsiError(RuntimeError):
    """A CUDA / cuBLAS / cuSOLVER / NCCL failure inside libchfsi."""


_vp = ctypes.c_void_p
_i = ctypes.c_int
_ll = ctypes.c_longlong
_d = ctypes.c_double
_c = ctypes.c_char
_pd = ctypes.POINTER(ctypes.c_double)
_pi = ctypes.POINTER(ctypes.c_int)

# name -> argtypes (restype is int unless listed in _RESTYPES)
_SIGNATURES = {
    "chfsi_version": [],
    "chfsi_last_error": [],
    "chfsi_launch_count": [],
    "chfsi_ctx_create": [_i, ctypes.POINTER(_vp)],
    "chfsi_ctx_destroy": [_vp],
    "chfsi_ctx_set_stream": [_vp, _vp],
    "chfsi_ctx_set_tiling": [_vp, _i, _i, _i],
    "chfsi_ctx_set_step_groups": [_vp, _i],
    "chfsi_ctx_set_step_warps": [_vp, _i],
    "chfsi_ctx_set_filter_chains": [_vp, _i],
    "chfsi_cheb_step_z": [_vp, _i, _i, _vp, _ll, _i, _vp, _ll, _vp, _ll, _vp, _ll, _d, _d, _d],
    "chfsi_cheb_step_rows_z": [_vp, _i, _i, _i, _vp, _ll, _i, _vp, _ll, _i, _i, _vp, _ll, _vp, _ll,
                               _vp, _ll, _d, _d, _d],
    "chfsi_cheb_step_rows_peers_z": [_vp, _i, _i, _i, _vp, _ll, _i, _vp, _ll, _i, _i, _vp, _ll, _vp,
                                     _ll, _vp, _ll, _d, _d, _d, ctypes.POINTER(_vp), _i],
    "chfsi_filter_coeffs": [_i, _d, _d, _d, _pd, _pd, _pd],
    "chfsi_filter_z": [_vp, _i, _i, _vp, _ll, _i, _vp, _ll, _vp, _vp, _ll, _i, _d, _d, _d,
                       ctypes.POINTER(_vp)],
    "chfsi_filter_degrees_z": [_vp, _i, _i, _vp, _ll, _i, _vp, _ll, _vp, _vp, _ll, _pi, _d, _d, _d,
                               ctypes.POINTER(_vp)],
    "chfsi_step_tiling": [_i, _i, _pi, _pi, _pi],
    "chfsi_set_complex_product": [_i],
    "chfsi_set_k1_slab": [_i],
    "chfsi_set_panel_kernels": [_i],
    "chfsi_debug_k1_trace": [ctypes.POINTER(ctypes.c_ulonglong), _i],
    "chfsi_lanczos_z": [_vp, _i, _i, _vp, _ll, _i, _vp, _vp, _pd, _pd, _pd, _pi],
    "chfsi_gemm_z": [_vp, _c, _c, _i, _i, _i, _d, _d, _vp, _ll, _vp, _ll, _d, _d, _vp, _ll],
    "chfsi_cgs_project_z": [_vp, _i, _i, _i, _vp, _ll, _vp, _ll, _vp],
    "chfsi_qr_orthonormalize_z": [_vp, _i, _i, _vp, _ll, _pi, _pi],
    "chfsi_ctx_set_qr_mode": [_vp, _i],
    "chfsi_ctx_set_qr_linear2": [_vp, _i],
    "chfsi_ctx_set_lanczos_mode": [_vp, _i],
    "chfsi_heevd_z": [_vp, _i, _vp, _ll, _vp],
    "chfsi_heev_rr_z": [_vp, _i, _vp, _ll, _vp, _d, _pi],
    "chfsi_colnorm_residual_z": [_vp, _i, _i, _vp, _ll, _vp, _ll, _vp, _vp],
    "chfsi_colnorm_residual_sq_z": [_vp, _i, _i, _vp, _ll, _vp, _ll, _vp, _vp],
    "chfsi_symmetrize_z": [_vp, _i, _vp, _ll],
    "chfsi_herm_defect_z": [_vp, _i, _vp, _ll, _pd, _pd],
    "chfsi_conj_z": [_vp, _i, _i, _vp, _ll],
    "chfsi_potrf_z": [_vp, _i, _vp, _ll, _pi],
    "chfsi_trsm_z": [_vp, _c, _c, _i, _i, _vp, _ll, _vp, _ll],
    "chfsi_to_standard_z": [_vp, _i, _vp, _ll, _vp, _ll, _i, _pi],
    "chfsi_to_standard_async_z": [_vp, _i, _vp, _ll, _vp, _ll, _i, _vp],
    "chfsi_to_standard_k1_z": [_vp, _i, _vp, _ll, _vp, _ll, _i, _vp, _vp],
    "chfsi_herm_defect_async_z": [_vp, _i, _vp, _ll, _vp],
    "chfsi_back_transform_z": [_vp, _i, _i, _vp, _ll, _vp, _ll],
}

FILTER_CB = ctypes.CFUNCTYPE(_i, _vp, _vp, _vp, _ll, _i, _i, _pi, _d, _d, _d, ctypes.POINTER(_vp))
FILL_CB = ctypes.CFUNCTYPE(_i, _vp, _vp, _ll, _i, _pi, _i)
ALLREDUCE_CB = ctypes.CFUNCTYPE(_i, _vp, _vp, _ll)
HP_CB = ctypes.CFUNCTYPE(_i, _vp, _vp, _vp, _ll, _i)
GATHER_CB = ctypes.CFUNCTYPE(_i, _vp, _vp, _ll, _i, ctypes.POINTER(_vp))


class LoopState(ctypes.Structure):
    """Mirror of `chfsi_loop` (include/chfsi.h): native ChFSI inner loop."""

    _fields_ = [
        ("n", _i), ("blk", _i), ("nev", _i), ("deg", _i), ("max_repeats", _i),
        ("adaptive", _i), ("deg_min", _i),
        ("tol", _d), ("rr_fast_tol", _d),
        ("H", _vp), ("ldh", _ll), ("conj_h", _i),
        ("bufs", _vp * 2), ("hp", _vp), ("hp_rot", _vp), ("locked", _vp), ("g", _vp),
        ("coef", _vp), ("ritz_d", _vp), ("res_d", _vp), ("perm_d", _vp), ("tail", _vp),
        ("row0", _i), ("n_local", _i), ("allreduce", ALLREDUCE_CB), ("hp_fn", HP_CB),
        ("gather", GATHER_CB),
        ("filter", FILTER_CB), ("fill", FILL_CB), ("user", _vp),
        ("win_a", _d), ("win_b", _d), ("win_scale_ref", _d),
        ("inner_loops", _i), ("nlocked", _i), ("pb", _i), ("off", _i), ("width", _i),
        ("converged", _i),
        ("last_rot_pb", _i), ("last_width", _i), ("last_nlock", _i),
        ("locked_vals", _pd), ("locked_res", _pd), ("locked_per_loop", _pi),
        ("ritz", _pd), ("res", _pd), ("degs", _pi),
        ("filtered_vectors", _ll), ("matvecs", _ll), ("residual_check_matvecs", _ll),
        ("filter_launches", _ll), ("rr_fast_eigs", _ll), ("filter_degree_sum", _ll),
        ("filter_flops", _d),
        ("t_filter", _d), ("t_ortho", _d), ("t_rr", _d),
        ("reuse_hp", _i), ("filter_k1_launches", _ll), ("filter_k1_flops", _d),
        ("qr_redone", _ll),
    ]


_SIGNATURES["chfsi_solve_loop_z"] = [_vp, ctypes.POINTER(LoopState)]
_SIGNATURES["chfsi_lanczos_rows_ws_bytes"] = [_i, _i]
_SIGNATURES["chfsi_lanczos_rows_z"] = [_vp, _i, _i, _vp, _ll, _i, _i, _i, _vp, _vp, _vp, ALLREDUCE_CB,
                                       GATHER_CB, _vp, _pd, _pd, _pd, _pi]

_RESTYPES = {"chfsi_last_error": ctypes.c_char_p, "chfsi_launch_count": ctypes.c_longlong,
             "chfsi_lanczos_rows_ws_bytes": ctypes.c_longlong}


def symbols():
    """Every entry point the binding expects (== the functions of include/chfsi.h)."""
    return sorted(_SIGNATURES)


_lib = None
_lib_lock = threading.Lock()


def lib():
    """Load libchfsi.so (once). Raises BackendUnavailable if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise BackendUnavailable(
                    f"{LIB_PATH} is not built; run `python -m paper_1206_3768_b200.csrc.build`")
            handle = ctypes.CDLL(LIB_PATH)
            for name, args in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = _RESTYPES.get(name, ctypes.c_int)
            _lib = handle
    return _lib


def last_error():
    msg = lib().chfsi_last_error()
    return msg.decode() if msg else ""


def check(status, what="", dead=None):
    """Map a CHFSI_E* status to the reference's exception classes."""
    if status == CHFSI_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == CHFSI_EINVAL:
        raise ValueError(msg)
    if status == CHFSI_ENOTPD:
        raise NotPositiveDefiniteError(msg)
    if status == CHFSI_ERANK:
        raise RankDeficientError(dead if dead is not None else ())
    if status == CHFSI_EEIG:
        raise EigenSolverError(msg)
    raise ChfsiError(f"status {status}: {msg}")


class _Ctx:
    def __init__(self, device):
        import torch

        self.device = device
        self.torch = torch
        h = _vp()
        check(lib().chfsi_ctx_create(device, ctypes.byref(h)), "chfsi_ctx_create")
        self.handle = h
        self._stream = None

    def bind_stream(self):
        """Point the context at torch's current stream on this device."""
        s = self.torch.cuda.current_stream(self.device).cuda_stream
        if s != self._stream:
            check(lib().chfsi_ctx_set_stream(self.handle, _vp(s)), "chfsi_ctx_set_stream")
            self._stream = s
        return self.handle


_ctxs = threading.local()


def ctx(device=None):
    """libchfsi context for (this thread, device, torch's current stream).

    One context per stream: contexts own cuBLAS/cuSOLVER handles and
    workspaces, so work issued concurrently on two streams (the sequence
    driver reduces problem l+1 while solving problem l) never shares them.
    """
    import torch

    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device visible: the ChFSI path runs only on the GPU")
    dev = torch.cuda.current_device() if device is None else int(device)
    stream = torch.cuda.current_stream(dev).cuda_stream
    table = getattr(_ctxs, "table", None)
    if table is None:
        table = _ctxs.table = {}
    c = table.get((dev, stream))
    if c is None:
        c = table[(dev, stream)] = _Ctx(dev)
    return c.bind_stream()


def dptr(t):
    return _vp(t.data_ptr())


def filter_coeffs(deg, a, b, scale_ref):
    """Host-side (c, alphas, betas) from the library (no GPU needed)."""
    al = np.zeros(deg)
    be = np.zeros(deg)
    c = ctypes.c_double()
    check(lib().chfsi_filter_coeffs(deg, a, b, scale_ref, ctypes.byref(c),
                                    al.ctypes.data_as(_pd), be.ctypes.data_as(_pd)),
          "chfsi_filter_coeffs")
    return c.value, al, be
