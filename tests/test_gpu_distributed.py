"""Row-sharded K1 on one B200 (the multi-GPU data path without NCCL).

Only one GPU is available to the test tiers, so the P ranks of the sharded
filter are emulated inside one process: every pseudo-rank runs its K1 row
shard (`chfsi_cheb_step_rows_z`, rank-blocked Y through the 3-D TMA map)
into its own block of ONE shared blocked buffer — which is exactly the
buffer state an in-place all-gather produces on a real rank. Kernels that
wait on one another are never co-scheduled (B200_PROFILING.md). The
collective itself is covered by tests/test_distributed_cpu.py (gloo).
"""

import numpy as np
import pytest
import torch

from oracle import chfsi_oracle as orc
from tests.golden.recipes import random_hermitian

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,w,world,deg,conj", [(300, 24, 2, 5, False), (1000, 97, 8, 4, True),
                                                (2048, 160, 4, 3, False), (777, 33, 3, 6, True)])
def test_emulated_row_sharded_filter_matches_single_gpu(n, w, world, deg, conj):
    import paper_1206_3768_b200 as pkg
    from paper_1206_3768_b200._device import Operator, to_fblock
    from paper_1206_3768_b200._lib import filter_coeffs
    from paper_1206_3768_b200.distributed import (RowPartition, blocked_empty, from_blocked,
                                                  gpu_row_step, to_blocked)

    rng = np.random.default_rng(n + world)
    h = random_hermitian(rng, n)
    y = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
    hd = torch.from_numpy(h).cuda()
    if conj:
        hd = hd.t().contiguous().t()  # column-major storage: the kernels read conj(H^T) = H
    op = Operator(hd)
    ev = np.linalg.eigvalsh(h)
    win = pkg.FilterWindow(a=float(ev[n // 3]), b=float(ev[-1]) + 0.2, scale_ref=float(ev[0]))
    c, al, be = filter_coeffs(deg, win.a, win.b, win.scale_ref)
    parts = [RowPartition(n, world, r) for r in range(world)]
    yd = to_fblock(y)
    bufs = [to_blocked(parts[0], yd, blocked_empty(parts[0], w, "cuda")),
            blocked_empty(parts[0], w, "cuda")]
    cur = 0
    for j in range(deg):
        nxt = 1 - cur
        for p in parts:  # every pseudo-rank writes its own block: the all-gather's result
            yprev = bufs[nxt][p.rank] if j > 0 else None
            gpu_row_step(op, p, bufs[cur], yprev, bufs[nxt][p.rank], w, al[j], c, be[j])
        cur = nxt
    out = from_blocked(parts[0], bufs[cur], torch.empty((w, n), dtype=torch.complex128,
                                                        device="cuda").t()).cpu().numpy()
    ref = orc.chebyshev_filter(h, y, deg, win.a, win.b, win.scale_ref)
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()
    single = pkg.chebyshev_filter(hd, yd, deg, win).cpu().numpy()
    assert np.abs(out - single).max() <= 1e-12 * np.abs(ref).max()


def test_row_sharded_filter_world1_uses_blocked_path():
    """RowShardedFilter without torch.distributed: one rank, blocked layout."""
    import paper_1206_3768_b200 as pkg
    from paper_1206_3768_b200._device import Operator, to_fblock
    from paper_1206_3768_b200.distributed import RowShardedFilter

    n, w, deg = 513, 40, 5
    rng = np.random.default_rng(3)
    h = random_hermitian(rng, n)
    y = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
    win = pkg.FilterWindow(a=0.0, b=float(np.linalg.eigvalsh(h)[-1]) + 0.1, scale_ref=-20.0)
    for chunks in (1, 3):
        out = RowShardedFilter(Operator(h), n, chunks=chunks).apply(to_fblock(y), deg, win)
        ref = orc.chebyshev_filter(h, y, deg, win.a, win.b, win.scale_ref)
        assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
