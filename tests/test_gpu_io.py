"""Device-side BASELINE generator vs the host generator.

The device path draws the same numpy Generator stream on the host and does
the O(n^3) algebra on the GPU, so it must reproduce the host sequence to
rounding (the host QR/GEMM and cuSOLVER/cuBLAS round differently).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,length", [(96, 3), (512, 4)])
def test_device_generator_matches_host(n, length):
    from paper_1206_3768_b200.sequence import iter_baseline_sequence

    host = list(iter_baseline_sequence(n, length, seed=0))
    dev = list(iter_baseline_sequence(n, length, seed=0, device="cuda:0"))
    assert [lab for lab, _, _ in dev] == list(range(1, length + 1))
    for (lh, ah, bh), (ld, ad, bd) in zip(host, dev):
        assert lh == ld
        assert ad.is_cuda and ad.is_contiguous() and ad.dtype == torch.complex128
        for x, y in ((ah, ad), (bh, bd)):
            y = y.cpu().numpy()
            assert np.abs(x - y).max() <= 1e-12 * np.abs(x).max()
            assert np.array_equal(y, y.conj().T)  # exactly Hermitian


def test_device_generator_feeds_the_solver():
    import paper_1206_3768_b200 as pkg

    cfg_b = pkg.BASELINE_CONFIGS["C1"]
    seq = list(pkg.iter_baseline_sequence(cfg_b.n, 2, seed=0, device="cuda:0"))
    res = pkg.solve_sequence(seq, pkg.ChfsiConfig(nev=cfg_b.nev, nex=cfg_b.nex, deg=cfg_b.deg))
    assert all(r.report.converged for r in res)


def test_lazy_device_generator_feeds_the_driver_directly():
    """The sequence driver stages problem l+1 on its side stream while it
    solves problem l; a LAZY device generator queues the work that writes
    A_{l+1}, B_{l+1} on the solver's stream inside next(). The staging must
    wait for it (the driver records an event after each next() and the side
    stream waits on it): fed the generator itself, the results are bitwise
    those of the materialised list."""
    import paper_1206_3768_b200 as pkg
    import torch

    cfg_b = pkg.BASELINE_CONFIGS["C1"]
    cfg = pkg.ChfsiConfig(nev=cfg_b.nev, nex=cfg_b.nex, deg=cfg_b.deg)
    listed = pkg.solve_sequence(list(pkg.iter_baseline_sequence(cfg_b.n, 4, seed=0, device="cuda:0")),
                                cfg)
    lazy = pkg.solve_sequence(pkg.iter_baseline_sequence(cfg_b.n, 4, seed=0, device="cuda:0"), cfg)
    assert len(lazy) == len(listed) == 4
    for a, b in zip(listed, lazy):
        assert a.report.locked_per_loop == b.report.locked_per_loop
        assert np.array_equal(a.values, b.values)
        assert torch.equal(a.solution.vectors, b.solution.vectors)
