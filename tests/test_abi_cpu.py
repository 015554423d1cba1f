"""CPU-side checks of the C-ABI boundary and the host logic (no GPU).

* libchfsi.so loads and exports every entry point include/chfsi.h declares;
* host-only entry points (filter coefficients, tile choice) agree with the
  oracle;
* the product path refuses to run without a GPU (no CPU fallback);
* host logic mirrors the reference (config resolution, window clamp,
  scalar response).
"""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

from oracle import chfsi_oracle as orc
from paper_1206_3768_b200 import _lib
from paper_1206_3768_b200.chfsi import (
    ChfsiConfig,
    FilterWindow,
    _safe_window,
    chebyshev_response,
)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "chfsi.h")).read()
    return sorted(set(re.findall(r"CHFSI_API\s+[\w\s\*]+?\b(chfsi_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == _lib.symbols()


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.chfsi_version() == 1


def test_library_is_sm100a_only():
    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob or b"sm_100" in blob


@pytest.mark.parametrize("deg,win", [(1, (0.3, 2.0, -1.1)), (16, (-0.4, 9.0, -0.9)),
                                     (36, (1.0, 5.0, -2.0))])
def test_filter_coefficients_match_oracle(deg, win):
    c, al, be = _lib.filter_coeffs(deg, *win)
    c0, al0, be0 = orc.filter_coefficients(deg, *win)
    assert c == c0
    assert np.array_equal(al, al0) and np.array_equal(be, be0)


def test_filter_coefficients_reject_bad_degree():
    with pytest.raises(ValueError):
        _lib.filter_coeffs(0, 0.0, 1.0, -1.0)


@pytest.mark.parametrize("n,w", [(512, 48), (2048, 160), (5000, 600), (20000, 3400), (97, 3)])
def test_tile_choice_is_valid(n, w):
    bm, bn, sp = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    assert _lib.lib().chfsi_step_tiling(n, w, ctypes.byref(bm), ctypes.byref(bn), ctypes.byref(sp)) == 0
    assert bm.value in (64, 128) and bn.value in (16, 32, 64) and sp.value == 0
    # never more padded columns than the narrowest tile would need
    assert -(-w // bn.value) * bn.value - w < max(bn.value, 16)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_product_path_fails_loudly_without_gpu():
    from paper_1206_3768_b200 import BackendUnavailable, chebyshev_filter

    h = np.eye(4, dtype=complex)
    with pytest.raises(BackendUnavailable):
        chebyshev_filter(h, np.ones((4, 1), dtype=complex), 3, FilterWindow(0.5, 2.0, 0.0))


@pytest.mark.parametrize("n,kw", [(512, dict(nev=32, nex=16)), (2048, dict(nev=128, nex=32)),
                                  (5000, dict(nev=500, nex=100)), (12000, dict(nev=1200, nex=200)),
                                  (20000, dict(nev=3000, nex=400)), (60, dict(nev=6)),
                                  (8, dict(nev=3))])
def test_config_resolution_matches_oracle(n, kw):
    cfg = ChfsiConfig(**kw)
    blk = kw["nev"] + kw.get("nex", 40)
    got = cfg.resolve(n)
    want = orc.resolve(n, kw["nev"], None if "nex" not in kw else blk)
    assert got == want


def test_config_validation():
    with pytest.raises(ValueError):
        ChfsiConfig(nev=0).resolve(10)
    with pytest.raises(ValueError):
        ChfsiConfig(nev=3, deg=0).resolve(10)
    with pytest.raises(ValueError):
        ChfsiConfig(nev=3, tol=0.0).resolve(10)
    with pytest.raises(ValueError):
        ChfsiConfig(nev=3, blk=10, nex=2)


@pytest.mark.parametrize("args", [(0.0, 1.0, 2.0), (0.0, -1.0, 2.0), (0.0, 3.0, 2.0),
                                  (5.0, 1.0, 2.0), (0.0, 1.0, np.inf)])
def test_safe_window_matches_oracle(args):
    w = _safe_window(*args)
    assert (w.a, w.b, w.scale_ref) == pytest.approx(orc.safe_window(*args), nan_ok=True)


def test_safe_window_nan_anchor_raises_like_reference():
    # chfsi.py:266-268 builds FilterWindow(nan+0.5, nan+1, nan), whose check raises
    with pytest.raises(ValueError):
        _safe_window(np.nan, 1.0, 2.0)


def test_window_validation():
    FilterWindow(a=1.0, b=2.0, scale_ref=0.0)
    with pytest.raises(ValueError):
        FilterWindow(a=2.0, b=1.0, scale_ref=0.0)
    with pytest.raises(ValueError):
        FilterWindow(a=1.0, b=2.0, scale_ref=1.5)


@pytest.mark.parametrize("deg", [1, 2, 7, 25, 120])
def test_response_matches_oracle(deg):
    win = FilterWindow(a=0.3, b=2.0, scale_ref=-1.1)
    lam = np.linspace(-1.1, 2.5, 77)
    np.testing.assert_allclose(chebyshev_response(lam, deg, win),
                               orc.chebyshev_response(lam, deg, 0.3, 2.0, -1.1), rtol=1e-14)
    assert abs(chebyshev_response(-1.1, deg, win)) == pytest.approx(1.0)
