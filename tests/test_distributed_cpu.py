"""Multi-process host logic of the row-sharded filter (gloo, world_size 2, CPU).

The production step is K1 on a B200 and the collective is NCCL; here the
step is a torch-CPU restatement of exactly the rows K1 computes
(chfsi.py:203-206 restricted to the rank's rows) and the collective is
gloo's all_gather_into_tensor. This checks the partition, the rank-blocked
layout, the in-place ping-pong, the per-step coefficients and the
column-chunk pipelining against the single-process oracle filter.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import chfsi_oracle as orc
from paper_1206_3768_b200.distributed import RowPartition, RowShardedFilter, from_blocked


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cpu_step(h, part):
    n = part.n

    def step(ycur_blk, yprev_slab, ynext_slab, w, alpha, c, beta):
        ycur = from_blocked(part, ycur_blk, torch.empty((w, n), dtype=torch.complex128).t())
        r0, rows = part.r0, part.rows
        if rows == 0:
            return
        prod = h[r0:r0 + rows, :] @ ycur
        own = ycur_blk[part.rank][:, :rows].t()
        res = alpha * (prod - c * own)
        if yprev_slab is not None:
            res = res - beta * yprev_slab[:, :rows].t()
        ynext_slab[:, :rows] = res.t()

    return step


def _worker(rank, world, port, n, w, deg, chunks, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        h = (g + g.conj().T) / 2
        y = rng.standard_normal((n, w)) + 1j * rng.standard_normal((n, w))
        ht = torch.from_numpy(h)
        yt = torch.from_numpy(np.asfortranarray(y))
        flt = RowShardedFilter(None, n, chunks=chunks)
        flt.step = _cpu_step(ht, flt.part)
        win = type("W", (), dict(a=-1.0, b=float(np.linalg.eigvalsh(h)[-1]) + 0.1, scale_ref=-2.5))
        out = flt.apply(yt, deg, win).numpy()
        if np.ndim(deg) == 0:
            ref = orc.chebyshev_filter(h, y, deg, win.a, win.b, win.scale_ref)
        else:  # per-column (adaptive) degrees, non-decreasing
            ref = orc.chebyshev_filter_degrees(h, y, deg, win.a, win.b, win.scale_ref)
        q.put((rank, float(np.abs(out - ref).max() / np.abs(ref).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,w,deg,chunks", [(64, 8, 5, 1), (101, 13, 7, 2), (150, 9, 4, 3),
                                            (90, 7, [1, 2, 2, 3, 5, 5, 6], 2)])
def test_row_sharded_filter_world2_matches_oracle(n, w, deg, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, w, deg, chunks, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert set(res) == {0, 1}
    for rank, err in res.items():
        assert err <= 1e-13, (rank, err)


@pytest.mark.parametrize("n,world", [(64, 2), (101, 2), (5000, 8), (12000, 8), (20000, 8), (17, 4)])
def test_row_partition_covers_rows(n, world):
    parts = [RowPartition(n, world, r) for r in range(world)]
    kblk = parts[0].kblk
    assert kblk % 16 == 0 and kblk * world >= n
    covered = []
    for p in parts:
        assert p.kblk == kblk
        covered.extend(range(p.r0, p.r0 + p.rows))
    assert covered == list(range(n))


# ---------------------------------------------- row-sharded reduction ---

class _HostLinalg:
    """Host restatement of the sharded reduction's local kernels (cuSOLVER
    potrf / cuBLAS ZTRSM on the GPU): numpy Cholesky, scipy triangular solve."""

    @staticmethod
    def potrf(b):
        return torch.from_numpy(np.asfortranarray(np.linalg.cholesky(np.asarray(b))))

    @staticmethod
    def trsm(l, x, conj_transpose=False):
        import scipy.linalg

        sol = scipy.linalg.solve_triangular(l.numpy(), x.numpy(), lower=True,
                                            trans="C" if conj_transpose else "N")
        x.copy_(torch.from_numpy(sol))
        return x


def _reduction_worker(rank, world, port, n, k, q):
    from paper_1206_3768_b200.distributed import RowComm, back_transform_rows, to_standard_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(11)
        g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        a = (g + g.conj().T) / 2
        c = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        b = np.eye(n) + c @ c.conj().T / (4 * n)
        b = (b + b.conj().T) / 2
        y = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
        comm = RowComm(n)
        op, l = to_standard_rows(torch.from_numpy(a), torch.from_numpy(b), comm, linalg=_HostLinalg)
        h_ref, l_ref = orc.to_standard(a, b)
        part = comm.part
        block = op.tensor.numpy()
        err_h = float(np.abs(block - h_ref[:, part.r0:part.r0 + part.rows]).max(initial=0.0))
        # the rows K1 reads: conj of the column block = H[rows, :]
        err_rows = float(np.abs(block.conj().T - h_ref[part.r0:part.r0 + part.rows, :])
                         .max(initial=0.0))
        herm = float(np.abs(block - h_ref[part.r0:part.r0 + part.rows, :].conj().T).max(initial=0.0))
        x = back_transform_rows(l, torch.from_numpy(np.asfortranarray(y)), comm,
                                linalg=_HostLinalg).numpy()
        err_x = float(np.abs(x - orc.back_transform(l_ref, y)).max())
        q.put((rank, dict(h=err_h, rows=err_rows, herm=herm, x=err_x, row0=op.row0,
                          nrows=op.rows, conj=op.conj, l=float(np.abs(l.numpy() - l_ref).max()))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,k,world", [(37, 5, 2), (50, 7, 3)])  # 50/3: rank 2 holds no rows
def test_row_sharded_reduction_matches_oracle(n, k, world):
    """to_standard_rows / back_transform_rows (reduction.py:102-134 split
    over the ranks): each rank's column block of H = L^-1 A L^-H (= its rows,
    conjugated) and the back-transformed block equal the oracle's, with two
    all-to-alls and one all-gather over gloo."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_reduction_worker, args=(r, world, port, n, k, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert set(res) == set(range(world))
    covered = 0
    for rank, r in sorted(res.items()):
        assert r["h"] <= 1e-12 and r["rows"] <= 1e-12 and r["herm"] <= 1e-12, (rank, r)
        assert r["x"] <= 1e-12 and r["l"] == 0.0 and r["conj"] == 1, (rank, r)
        assert r["row0"] == covered
        covered += r["nrows"]
    assert covered == n
