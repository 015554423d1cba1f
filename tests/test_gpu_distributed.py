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


@pytest.mark.parametrize("n,w,world,conj", [(300, 24, 2, False), (777, 33, 3, True), (2048, 96, 8, False)])
def test_fused_allgather_epilogue_stores_to_every_peer(n, w, world, conj):
    """K1 with the fused all-gather: each pseudo-rank's epilogue stores its
    row slab into its own blocked buffer AND at the same position of every
    'peer' buffer (here other allocations of this process standing in for
    the peers' IPC-mapped buffers). After one step of every rank, all P
    buffers must hold the same full result, equal to the unfused path."""
    import ctypes

    import paper_1206_3768_b200 as pkg  # noqa: F401
    from paper_1206_3768_b200 import _lib
    from paper_1206_3768_b200._device import Operator, to_fblock
    from paper_1206_3768_b200.distributed import RowPartition, blocked_empty, gpu_row_step, to_blocked

    rng = np.random.default_rng(n * world + w)
    h = random_hermitian(rng, n)
    y = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
    hd = torch.from_numpy(h).cuda()
    if conj:
        hd = hd.t().contiguous().t()
    op = Operator(hd)
    parts = [RowPartition(n, world, r) for r in range(world)]
    ycur = to_blocked(parts[0], to_fblock(y), blocked_empty(parts[0], w, "cuda"))
    # unfused reference: every rank writes its slab of one shared buffer
    ref = blocked_empty(parts[0], w, "cuda")
    for p in parts:
        gpu_row_step(op, p, ycur, None, ref[p.rank], w, 0.7, -0.3, 0.0)
    # fused: rank p owns `outs[p]`; its epilogue also stores into outs[q != p]
    outs = [blocked_empty(parts[0], w, "cuda") for _ in range(world)]
    for p in parts:
        mine = outs[p.rank][p.rank]
        peers = [outs[q][p.rank].data_ptr() for q in range(world) if q != p.rank]
        gpu_row_step(op, p, ycur, None, mine, w, 0.7, -0.3, 0.0, peers=peers)
    torch.cuda.synchronize()
    for q in range(world):
        assert torch.equal(outs[q], ref), q
    # argument checks of the C-ABI
    L = _lib.lib()
    arr = (ctypes.c_void_p * 8)(*([outs[0].data_ptr()] * 8))
    st = L.chfsi_cheb_step_rows_peers_z(_lib.ctx(), n, parts[0].rows, w, ctypes.c_void_p(hd.data_ptr()),
                                        op.ld, op.conj, _lib.dptr(ycur), 0, parts[0].kblk, world,
                                        _lib.dptr(ycur[0]), parts[0].kblk, None, parts[0].kblk,
                                        _lib.dptr(outs[0][0]), parts[0].kblk, 1.0, 0.0, 0.0, arr, 8)
    assert st == -1  # more than 7 peers: CHFSI_EINVAL


def test_fused_sharded_filter_world1_symmetric_memory():
    """The symmetric-memory plumbing of the fused all-gather (allocation,
    IPC rendezvous, cross-rank barrier, slab addressing) in a 1-rank NCCL
    group: the filter must match the oracle. (A real multi-rank run needs
    several GPUs; the peer-store arithmetic is covered above.)"""
    import os
    import socket

    import torch.distributed as dist

    import paper_1206_3768_b200 as pkg
    from paper_1206_3768_b200._device import Operator, to_fblock
    from paper_1206_3768_b200.distributed import RowShardedFilter

    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n, w, deg = 700, 40, 5
        rng = np.random.default_rng(11)
        h = random_hermitian(rng, n)
        y = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
        win = pkg.FilterWindow(a=0.0, b=float(np.linalg.eigvalsh(h)[-1]) + 0.1, scale_ref=-25.0)
        flt = RowShardedFilter(Operator(h), n, chunks=2, fused=True, max_cols=64)
        assert flt.symm is not None
        ref = orc.chebyshev_filter(h, y, deg, win.a, win.b, win.scale_ref)
        for _ in range(2):  # buffers are reused across calls
            out = flt.apply(to_fblock(y), deg, win).cpu().numpy()
            assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()
        degs = [2, 2, 3] + [5] * (w - 3)
        out = flt.apply(to_fblock(y), degs, win).cpu().numpy()
        refd = orc.chebyshev_filter_degrees(h, y, degs, win.a, win.b, win.scale_ref)
        assert np.abs(out - refd).max() <= 1e-12 * np.abs(refd).max()
    finally:
        dist.destroy_process_group()
