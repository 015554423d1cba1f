"""The row-sharded ChFSI loop (chfsi_solve(shard=...)) with P
emulated ranks on one B200.

Each rank is a host thread with its own CUDA stream and libchfsi context,
holding only its rows of every n x w block; the collectives (all-reduce of
the partial Grams / residual norms, row gathers) go through the host with a
thread barrier, in rank order — no kernel ever waits on another rank's
kernel (B200_PROFILING.md), the synchronisation is host-side. The filter
and H*P are computed on the gathered panel (their row-sharded K1 and fused
all-gather are covered by tests/test_gpu_distributed.py). The result must
equal the single-GPU solve: this checks the local-row bookkeeping of the
native loop, the distributed CGS / Cholesky-QR2 / Rayleigh-Ritz with
all-reduced partial products, locking, the tail and the gathers.

The sequence tests run the production RowComm operators instead (only the
NCCL calls replaced by the host hub): the row-sharded reduction (each rank
holds only its row block of H, two all-to-alls), row K1 filter steps on
the rank-blocked panel, the row Lanczos and the column-split back-transform.
"""

import threading

import numpy as np
import pytest
import torch

from tests.conftest import subspace_sines
from tests.golden.recipes import random_hermitian

pytestmark = pytest.mark.gpu


class _Hub:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def exchange(self, rank, value, reduce=False):
        self.slots[rank] = value
        self.barrier.wait()
        if reduce:
            res = self.slots[0].clone()
            for v in self.slots[1:]:
                res += v
        else:
            res = list(self.slots)
        self.barrier.wait()
        return res


class ThreadComm:
    """distributed.RowComm stand-in: P threads of one process, host collectives."""

    def __init__(self, n, world, rank, hub):
        from paper_1206_3768_b200.distributed import RowPartition

        self.part = RowPartition(n, world, rank)
        self.hub = hub

    def allreduce_(self, t):
        torch.cuda.current_stream().synchronize()
        total = self.hub.exchange(self.part.rank, t.detach().cpu(), reduce=True)
        t.copy_(total.to(t.device))

    def gather_rows(self, local, full):
        torch.cuda.current_stream().synchronize()
        parts = self.hub.exchange(self.part.rank, local.detach().cpu())
        full.copy_(torch.cat(parts, 0).to(full.device))
        return full

    def _full(self, local):
        from paper_1206_3768_b200._device import fblock

        return self.gather_rows(local, fblock(self.part.n, local.shape[1], local.device))

    def filter_local(self, op, blk, panel_local, deg, window, out_local):
        import paper_1206_3768_b200 as pkg

        res = pkg.chebyshev_filter(op.tensor, self._full(panel_local), deg, window)
        out_local.copy_(res[self.part.r0:self.part.r0 + self.part.rows])
        return out_local

    def hp_local(self, op, panel_local, out_local):
        from paper_1206_3768_b200.reduction import _apply

        hp = _apply(op.tensor, self._full(panel_local))
        out_local.copy_(hp[self.part.r0:self.part.r0 + self.part.rows])
        return out_local


def _run_ranks(world, fn):
    hub = _Hub(world)
    out, errs = [None] * world, [None] * world

    def worker(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = fn(r, hub)
                torch.cuda.current_stream().synchronize()
        except BaseException as exc:  # noqa: BLE001
            errs[r] = exc
            hub.barrier.abort()

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    for e in errs:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    assert all(o is not None for o in out)
    return out


@pytest.mark.parametrize("n,nev,blk,world,adaptive", [(400, 12, 24, 2, False), (777, 20, 36, 3, False),
                                                      (512, 16, 32, 4, True)])
def test_row_sharded_loop_matches_single_gpu(n, nev, blk, world, adaptive):
    import paper_1206_3768_b200 as pkg

    rng = np.random.default_rng(n + world)
    h = random_hermitian(rng, n)
    cfg = pkg.ChfsiConfig(nev=nev, blk=blk, deg=10, adaptive_degree=adaptive)
    ref, rrep = pkg.chfsi_solve(h, cfg, rng=5)
    hd = torch.from_numpy(h).cuda()

    def solve(r, hub):
        return pkg.chfsi_solve(hd, cfg, rng=5, shard=ThreadComm(n, world, r, hub))

    outs = _run_ranks(world, solve)
    for sol, rep in outs:
        assert rep.converged and rep.inner_loops == rrep.inner_loops
        assert rep.locked_per_loop == rrep.locked_per_loop
        assert np.abs(sol.values - ref.values).max() <= 1e-11 * np.abs(ref.values).max()
        assert rep.final_residuals.max() <= cfg.tol
        v = sol.vectors.cpu().numpy()
        assert v.shape == (n, nev)
        assert subspace_sines(ref.vectors.cpu().numpy(), v).max() <= 1e-9
    # every rank returns the same bytes
    for sol, _ in outs[1:]:
        assert np.array_equal(sol.values, outs[0][0].values)
        assert torch.equal(sol.vectors, outs[0][0].vectors)


def test_row_sharded_sequence_warm_starts_from_local_tails():
    import paper_1206_3768_b200 as pkg

    cfg_b = pkg.BASELINE_CONFIGS["C1"]
    cfg = pkg.ChfsiConfig(nev=cfg_b.nev, nex=cfg_b.nex, deg=cfg_b.deg)
    seq = list(pkg.iter_baseline_sequence(cfg_b.n, 3, seed=0))
    ref = pkg.solve_sequence(seq, cfg, seed=0)
    world = 2

    def run(r, hub):
        return pkg.solve_sequence(seq, cfg, seed=0, shard=_thread_row_comm(cfg_b.n, world, r, hub))

    outs = _run_ranks(world, run)
    for res in outs:
        for g, f in zip(res, ref):
            assert g.report.inner_loops == f.report.inner_loops
            assert np.abs(g.values - f.values).max() <= 1e-11 * np.abs(f.values).max()
            assert g.report.tail_vectors.shape[0] < cfg_b.n  # local rows only


def _thread_row_comm(n, world, rank, hub):
    """distributed.RowComm with host-mediated collectives among threads: the
    production row-sharded operators (RowOperator, row K1 steps on rank-
    blocked panels, row Lanczos) with the NCCL calls replaced by `hub`."""
    from paper_1206_3768_b200.distributed import RowComm, RowPartition, RowShardedFilter

    class ThreadRowComm(RowComm):
        def __init__(self):
            self.group, self.chunks, self._filters = None, 1, {}
            self.part = RowPartition(n, world, rank)

        def _sync(self):
            torch.cuda.current_stream().synchronize()

        def allreduce_(self, t):
            self._sync()
            t.copy_(hub.exchange(rank, t.detach().cpu(), reduce=True).to(t.device))

        def alltoall_blocks(self, send):
            self._sync()
            every = hub.exchange(rank, send.detach().cpu())
            return torch.stack([every[q][rank] for q in range(world)]).to(send.device)

        def allgather_blocks(self, mine):
            self._sync()
            return torch.stack(hub.exchange(rank, mine.detach().cpu())).to(mine.device)

        def _allgather_slabs(self, buf, async_op=False):
            self._sync()
            slabs = hub.exchange(rank, buf[rank].detach().cpu())
            for q, sl in enumerate(slabs):
                if q != rank:
                    buf[q].copy_(sl.to(buf.device))
            return None

        def gather_blocked(self, local, blocked):
            if self.part.rows:
                blocked[rank, :, : self.part.rows].copy_(local.t())
            self._allgather_slabs(blocked)
            return blocked

        def filter(self, op, blk):
            key = (id(op.tensor), op.tensor.data_ptr(), blk)
            f = self._filters.get(key)
            if f is None:
                f = RowShardedFilter(op, n, allgather=self._allgather_slabs, fused=False)
                f.part = self.part
                self._filters[key] = f
            return f

    return ThreadRowComm()


@pytest.mark.parametrize("n,world,adaptive", [(512, 2, False), (333, 3, False), (400, 2, True)])
def test_row_sharded_sequence_matches_single_gpu(n, world, adaptive):
    """The sharded sequence driver (solve_sequence(shard=...)): per problem
    the row-sharded reduction leaves each emulated rank only its row block of
    H (two all-to-alls), the solve runs the row-sharded loop (row Lanczos,
    row K1 filter steps on the rank-blocked panel, distributed QR / RR), and
    the back-transform splits the columns — equal to the single-GPU
    sequence: same loops and locking, eigenvalues to 1e-11, the standard and
    generalized eigenspaces to 1e-9, identical bytes on every rank."""
    import paper_1206_3768_b200 as pkg

    nev, nex = 16, 16
    cfg = pkg.ChfsiConfig(nev=nev, nex=nex, deg=10, adaptive_degree=adaptive)
    seq = list(pkg.iter_baseline_sequence(n, 3, seed=1))
    ref = pkg.solve_sequence(seq, cfg, seed=0, keep_standard=True)

    def run(r, hub):
        comm = _thread_row_comm(n, world, r, hub)
        res = pkg.solve_sequence(seq, cfg, seed=0, keep_standard=True, shard=comm)
        held = [comm.part.r0, comm.part.rows]
        return res, held

    outs = _run_ranks(world, run)
    for res, held in outs:
        for a, b in zip(ref, res):
            assert b.report.converged
            assert a.report.inner_loops == b.report.inner_loops
            assert a.report.locked_per_loop == b.report.locked_per_loop
            assert np.abs(a.values - b.values).max() <= 1e-11 * np.abs(a.values).max()
            assert b.report.final_residuals.max() <= cfg.tol
            assert subspace_sines(a.standard_vectors.cpu().numpy(),
                                  b.standard_vectors.cpu().numpy()).max() <= 1e-9
            xa, xb = a.solution.vectors.cpu().numpy(), b.solution.vectors.cpu().numpy()
            assert b.solution.form == "generalized" and xb.shape == xa.shape
            # B-orthonormal generalized vectors: compare spans through B
            qa, _ = np.linalg.qr(xa)
            qb, _ = np.linalg.qr(xb)
            assert subspace_sines(qa, qb).max() <= 1e-9
    covered = sorted(tuple(h) for _, h in outs)
    assert sum(r for _, r in covered) == n
    for res, _ in outs[1:]:
        for a, b in zip(outs[0][0], res):
            assert np.array_equal(a.values, b.values)
            assert torch.equal(a.solution.vectors, b.solution.vectors)
