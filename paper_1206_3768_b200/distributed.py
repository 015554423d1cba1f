"""Row-sharded Chebyshev filter across GPUs (`north_star` (4)).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch). Rank p
owns rows [p*kblk, (p+1)*kblk) of the filter output; every step

    Y_next[rows_p] = alpha (H[rows_p, :] Y_cur - c Y_cur[rows_p]) - beta Y_prev[rows_p]

is one K1 launch over the shard (`chfsi_cheb_step_rows_z`), followed by an
in-place NCCL all-gather of the row slabs so every rank holds the full
Y_next for the next step. The full block lives in a *rank-blocked* layout
— block q = rows [q*kblk, (q+1)*kblk), column-major inside, zero padding
rows — which is exactly what an in-place all-gather of the per-rank slabs
produces, and K1 reads it directly through a 3-D TMA map: no pack/unpack
between steps. The step is column-chunked (`chunks`): the all-gather of
chunk c runs on a communication stream while K1 computes chunk c+1, so the
NVLink transfer overlaps the tensor-core work.

The reference has no parallel code (one process, BLAS threads);
the result is identical to the single-GPU filter up to the summation order
of the GEMM (the K split differs), i.e. rounding.

The local step and the collective are injectable so the host logic
(partition, ping-pong, coefficients, chunking, all-gather order) is tested
with the gloo backend on CPU (tests/test_distributed_cpu.py).
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

from ._device import Operator
from ._lib import check, ctx, dptr, filter_coeffs, lib

__all__ = ["RowPartition", "RowShardedFilter", "RowComm", "RowOperator", "gpu_row_step",
           "to_standard_rows", "back_transform_rows"]

BK = 32  # K1's deepest k-slab (32 complex): blocked rows per rank are a multiple of it


class RowPartition:
    """Uniform 1-D row blocks: rank p owns [p*kblk, min(n, (p+1)*kblk))."""

    def __init__(self, n, world, rank):
        if world < 1 or not 0 <= rank < world:
            raise ValueError("bad world/rank")
        self.n, self.world, self.rank = n, world, rank
        self.kblk = max(BK, int(math.ceil(math.ceil(n / world) / BK)) * BK)
        self.r0 = min(n, rank * self.kblk)
        self.rows = max(0, min(n, self.r0 + self.kblk) - self.r0)

    def block_range(self, q):
        r0 = min(self.n, q * self.kblk)
        return r0, max(0, min(self.n, r0 + self.kblk) - r0)


def blocked_empty(part, w, device, dtype=torch.complex128):
    """Zero-initialised rank-blocked buffer [world][w][kblk] (padding rows stay 0)."""
    return torch.zeros((part.world, w, part.kblk), dtype=dtype, device=device)


def to_blocked(part, y, out):
    """Full column-major n x w -> rank-blocked buffer."""
    for q in range(part.world):
        r0, rows = part.block_range(q)
        if rows:
            out[q, :, :rows].copy_(y[r0:r0 + rows, :].t())
    return out


def from_blocked(part, buf, out):
    """Rank-blocked buffer -> full column-major n x w (out is an F-block view)."""
    for q in range(part.world):
        r0, rows = part.block_range(q)
        if rows:
            out[r0:r0 + rows, :].copy_(buf[q, :, :rows].t())
    return out


def gpu_row_step(op, part, ycur_blk, yprev_slab, ynext_slab, w, alpha, c, beta, peers=None):
    """K1 over this rank's rows (libchfsi); slabs are [w][kblk] views of
    the rank's block (column-major, ld kblk). ``peers``: device addresses of
    the same slab in the other ranks' buffers (mapped into this process) —
    the fused all-gather, K1's epilogue storing every tile to them too."""
    if part.rows == 0:
        return
    import ctypes

    h_rows = op.row_ptr(part.r0, part.rows)
    ycur_rows = ycur_blk[part.rank]
    args = (ctx(), part.n, part.rows, w, ctypes_ptr(h_rows), op.ld, op.conj, dptr(ycur_blk), 0,
            part.kblk, part.world, dptr(ycur_rows), part.kblk,
            None if yprev_slab is None else dptr(yprev_slab), part.kblk, dptr(ynext_slab),
            part.kblk, alpha, c, beta)
    if peers:
        arr = (ctypes.c_void_p * len(peers))(*peers)
        check(lib().chfsi_cheb_step_rows_peers_z(*args, arr, len(peers)),
              "sharded chebyshev step (fused all-gather)")
    else:
        check(lib().chfsi_cheb_step_rows_z(*args), "sharded chebyshev step")


class SymmetricBlocks:
    """Fused-all-gather storage: one symmetric-memory allocation per rank
    (torch.distributed._symmetric_memory, CUDA IPC over NVLink) holding the
    ping-pong rank-blocked buffers of every column group, identical layout on
    all ranks, so a slab's peer address is the peer's base + the same offset.
    `barrier()` is the cross-rank device barrier that orders filter steps."""

    def __init__(self, part, cols, group, device):
        import torch.distributed._symmetric_memory as symm

        self.part = part
        self.elems = 2 * part.world * cols * part.kblk  # two ping-pong slots
        self.buf = symm.empty(self.elems, dtype=torch.complex128, device=device)
        self.handle = symm.rendezvous(self.buf, group if group is not None else dist.group.WORLD)
        self.base = self.buf.data_ptr()
        self.peer_bases = [int(self.handle.buffer_ptrs[q]) for q in range(part.world)]
        self.cols = cols

    def views(self, groups):
        """[(slot0, slot1)] blocked views [world][wg][kblk] per column group."""
        out, off = [], 0
        span = self.part.world * self.part.kblk
        for j0, j1, _ in groups:
            wg = j1 - j0
            pair = []
            for s in range(2):
                start = s * self.part.world * self.cols * self.part.kblk + off
                pair.append(self.buf[start:start + wg * span].view(self.part.world, wg,
                                                                   self.part.kblk))
            out.append(pair)
            off += wg * span
        return out

    def peers_of(self, slab):
        """Device addresses of `slab` (a view into this rank's buffer) on the other ranks."""
        off = slab.data_ptr() - self.base
        return [self.peer_bases[q] + off for q in range(self.part.world) if q != self.part.rank]

    def barrier(self):
        self.handle.barrier(channel=0)


_SYMM_CACHE = {}


def fused_available(group=None):
    """NCCL world > 1 with torch symmetric memory (CUDA IPC peers)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return False
    if dist.get_backend(group) != "nccl":
        return False
    try:
        import torch.distributed._symmetric_memory  # noqa: F401
    except ImportError:
        return False
    return True


def ctypes_ptr(addr):
    import ctypes

    return ctypes.c_void_p(addr)


def nccl_allgather(buf, part, group=None, async_op=False):
    """In-place all-gather of the rank slabs of a blocked buffer [world][w][kblk]."""
    if part.world == 1:
        return None
    flat = buf.view(-1)
    chunk = flat.numel() // part.world
    mine = flat[part.rank * chunk:(part.rank + 1) * chunk]
    if dist.get_backend(group) != "nccl":  # in-place aliasing is an NCCL guarantee only
        mine = mine.clone()
    return dist.all_gather_into_tensor(flat, mine, group=group, async_op=async_op)


class RowShardedFilter:
    """Degree-`deg` filter (chfsi.py:179-208) with the row-sharded step.

    Columns are independent through the whole recurrence (chfsi.py:203-206),
    so the block is split into `chunks` column groups, each with its own pair
    of blocked buffers: the all-gather of group c (asynchronous, on the
    collective stream) overlaps K1 on group c+1, and step j+1 of group c only
    waits for group c's all-gather of step j.

    `step(ycur_blk, yprev_slab, ynext_slab, w, alpha, c, beta)` computes this
    rank's rows; `allgather(buf, async_op)` makes the blocked buffer full on
    every rank and may return a handle with `.wait()`. Defaults: K1 through
    libchfsi and NCCL.
    """

    def __init__(self, op, n, group=None, step=None, allgather=None, chunks=1, fused=None,
                 max_cols=None):
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.part = RowPartition(n, world, rank)
        self.op = op
        self.chunks = max(1, int(chunks))
        # fused all-gather: K1's epilogue stores each tile into every peer's
        # buffer (NVLink P2P, symmetric memory); default on for NCCL worlds > 1
        if fused is None:
            fused = step is None and allgather is None and fused_available(group)
        self.symm = None
        if fused:
            if max_cols is None:
                raise ValueError("the fused all-gather needs max_cols (the widest panel)")
            dev = op.tensor.device if op is not None else torch.device("cuda")
            key = (id(group), str(dev), n, world, int(max_cols))
            self.symm = _SYMM_CACHE.get(key)
            if self.symm is None:  # collective allocation + IPC rendezvous: once per shape
                self.symm = _SYMM_CACHE[key] = SymmetricBlocks(self.part, int(max_cols), group, dev)
        self.step = step or (lambda yc, yp, yn, w, a, c, b: gpu_row_step(op, self.part, yc, yp, yn,
                                                                        w, a, c, b))
        self.allgather = allgather or (lambda buf, async_op=False: nccl_allgather(
            buf, self.part, self.group, async_op))

    def apply(self, y, deg, window, out=None):
        """Filter the full block y (n x w, replicated on all ranks); returns
        the full filtered block (replicated), column-major. ``deg`` is one
        degree, or non-decreasing per-column degrees (adaptive mode): the
        columns then form groups of equal degree that leave the shared
        recurrence as their degree is reached."""
        part = self.part
        n, w = y.shape
        if n != part.n:
            raise ValueError("operator/block shapes do not conform")
        dev = y.device
        if np.ndim(deg) == 0:
            dmax = int(deg)
            nchunks = 1 if part.world == 1 else min(self.chunks, w)  # nothing to overlap alone
            edges = np.linspace(0, w, nchunks + 1).astype(int)
            groups = [(int(edges[k]), int(edges[k + 1]), dmax) for k in range(len(edges) - 1)
                      if edges[k + 1] > edges[k]]
        else:
            degs = [int(d) for d in deg]
            if len(degs) != w or min(degs) < 1 or any(b < a for a, b in zip(degs, degs[1:])):
                raise ValueError("per-column degrees must be >= 1 and non-decreasing")
            dmax = degs[-1]
            groups, j0 = [], 0
            for j in range(1, w + 1):
                if j == w or degs[j] != degs[j0]:
                    groups.append((j0, j, degs[j0]))
                    j0 = j
        c, al, be = filter_coeffs(dmax, float(window.a), float(window.b), float(window.scale_ref))
        if self.symm is not None:
            return self._apply_fused(y, groups, dmax, c, al, be, out)
        bufs = [[to_blocked(part, y[:, j0:j1], blocked_empty(part, j1 - j0, dev)),
                 blocked_empty(part, j1 - j0, dev)] for j0, j1, _ in groups]
        pending = [None] * len(groups)
        cur = [0] * len(groups)
        for j in range(dmax):
            for g, (j0, j1, dg) in enumerate(groups):
                if j >= dg:
                    continue  # this group reached its degree
                if pending[g] is not None:
                    pending[g].wait()  # step j of group g needs its step j-1 all-gather
                    pending[g] = None
                nxt = 1 - cur[g]
                yprev = bufs[g][nxt][part.rank] if j > 0 else None
                self.step(bufs[g][cur[g]], yprev, bufs[g][nxt][part.rank], j1 - j0, al[j], c, be[j])
                pending[g] = self.allgather(bufs[g][nxt], async_op=True)
                cur[g] = nxt
        for h in pending:
            if h is not None:
                h.wait()
        if out is None:
            out = torch.empty((w, n), dtype=y.dtype, device=dev).t()
        for g, (j0, j1, _) in enumerate(groups):
            from_blocked(part, bufs[g][cur[g]], out[:, j0:j1])
        return out

    def _apply_fused(self, y, groups, dmax, c, al, be, out):
        """Every step: K1 over this rank's rows of each column group, its
        epilogue storing the tiles into all ranks' next buffers; then one
        cross-rank barrier (all slabs landed before anyone reads them)."""
        part, symm = self.part, self.symm
        n, w = y.shape
        if w > symm.cols:
            raise ValueError(f"panel wider ({w}) than the symmetric buffers ({symm.cols})")
        pairs = symm.views(groups)
        for (j0, j1, _), pair in zip(groups, pairs):
            pair[0].zero_()  # K padding rows must read as 0; peers write real rows only
            pair[1].zero_()
            to_blocked(part, y[:, j0:j1], pair[0])
        symm.barrier()  # every rank's start block is in place before step 0 reads it
        cur = [0] * len(groups)
        for j in range(dmax):
            for g, (j0, j1, dg) in enumerate(groups):
                if j >= dg:
                    continue
                nxt = 1 - cur[g]
                yprev = pairs[g][nxt][part.rank] if j > 0 else None
                ynext = pairs[g][nxt][part.rank]
                gpu_row_step(self.op, part, pairs[g][cur[g]], yprev, ynext, j1 - j0, al[j], c,
                             be[j], peers=symm.peers_of(ynext))
                cur[g] = nxt
            symm.barrier()
        if out is None:
            out = torch.empty((w, n), dtype=y.dtype, device=y.device).t()
        for g, (j0, j1, _) in enumerate(groups):
            from_blocked(part, pairs[g][cur[g]], out[:, j0:j1])
        return out


# ------------------------------------------------------ row-sharded loop ---

class RowComm:
    """Collectives of the row-sharded ChFSI loop (chfsi_solve(shard=...)):
    every n x w block lives as this rank's rows; products over rows are
    summed with `allreduce_`, panels are made whole with `gather_rows` for
    the filter and H*P (both run as row-sharded K1 steps). NCCL over
    torch.distributed by default; `tests/test_gpu_distributed.py` drives the
    same interface with host-mediated collectives among threads."""

    def __init__(self, n, group=None, chunks=2):
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.part = RowPartition(n, world, rank)
        self.chunks = chunks
        self._filters = {}

    # -- collectives
    def allreduce_(self, t):
        """In-place sum over the ranks (identical bytes everywhere)."""
        if self.part.world > 1:
            dist.all_reduce(t, group=self.group)

    def alltoall_blocks(self, send):
        """send [world][...] -> recv with recv[q] = rank q's send[this rank]."""
        if self.part.world == 1:
            return send.clone()
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv.view(-1), send.view(-1), group=self.group)
        return recv

    def allgather_blocks(self, mine):
        """[...] on every rank -> [world][...] (rank q's tensor at index q)."""
        if self.part.world == 1:
            return mine.unsqueeze(0).clone()
        out = torch.empty((self.part.world,) + tuple(mine.shape), dtype=mine.dtype,
                          device=mine.device)
        dist.all_gather_into_tensor(out.view(-1), mine.contiguous().view(-1), group=self.group)
        return out

    def gather_blocked(self, local, blocked):
        """Local rows (nl x w F-block) -> full rank-blocked buffer on every rank."""
        part = self.part
        if part.rows:
            blocked[part.rank, :, :part.rows].copy_(local.t())
        nccl_allgather(blocked, part, self.group)
        return blocked

    def gather_rows(self, local, full):
        """Local rows -> full n x w F-block on every rank."""
        w = local.shape[1]
        blocked = self.gather_blocked(local, blocked_empty(self.part, w, local.device))
        return from_blocked(self.part, blocked, full)

    # -- sharded operators
    def filter(self, op, blk):
        key = (id(op.tensor), op.tensor.data_ptr(), blk)
        f = self._filters.get(key)
        if f is None:
            f = self._filters[key] = RowShardedFilter(op, self.part.n, group=self.group,
                                                      chunks=self.chunks, max_cols=blk)
        return f

    def filter_local(self, op, blk, panel_local, deg, window, out_local):
        """Filter the distributed panel; this rank's rows of the result."""
        n, w = self.part.n, panel_local.shape[1]
        full = torch.empty((w, n), dtype=panel_local.dtype, device=panel_local.device).t()
        self.gather_rows(panel_local, full)
        res = self.filter(op, blk).apply(full, deg, window)
        part = self.part
        out_local.copy_(res[part.r0:part.r0 + part.rows])
        return out_local

    def hp_local(self, op, panel_local, out_local):
        """This rank's rows of H * P (one row-sharded K1 product step)."""
        part, w = self.part, panel_local.shape[1]
        blocked = self.gather_blocked(panel_local, blocked_empty(part, w, panel_local.device))
        slab = torch.empty((w, part.kblk), dtype=panel_local.dtype, device=panel_local.device)
        gpu_row_step(op, part, blocked, None, slab, w, 1.0, 0.0, 0.0)
        out_local.copy_(slab[:, :part.rows].t())
        return out_local


def lanczos_rows(comm, op, k, q0):
    """Row-sharded k-step Lanczos (chfsi.py:125-162) over `comm` (a RowComm
    or a stand-in): returns (alphas, betas, beta_last, steps) on the host,
    identical on every rank. q0: the full start vector (numpy, replicated)."""
    import ctypes

    from ._device import fblock

    part = comm.part
    n, nl = part.n, part.rows
    dev = op.tensor.device
    k = min(k, n)
    nbytes = int(lib().chfsi_lanczos_rows_ws_bytes(nl, k))
    ws = torch.zeros((nbytes + 7) // 8, dtype=torch.float64, device=dev)
    basis = fblock(nl, k, dev)
    qfull = torch.empty((1, n), dtype=torch.complex128, device=dev).t()
    q0d = torch.from_numpy(np.ascontiguousarray(q0)).to(dev)
    err = []

    def allreduce(user, buf, count):
        try:
            off = (buf - ws.data_ptr()) // 8
            if not (0 <= off and off + count <= ws.numel() and ws.data_ptr() + 8 * off == buf):
                raise ValueError("allreduce pointer outside the Lanczos workspace")
            comm.allreduce_(ws[off:off + count])
            return 0
        except BaseException as exc:  # noqa: BLE001
            err.append(exc)
            return -1

    def gather(user, local, ld, width, out):
        try:
            j = (local - basis.data_ptr()) // (16 * nl)
            comm.gather_rows(basis[:, j:j + 1], qfull)
            out[0] = qfull.data_ptr()
            return 0
        except BaseException as exc:  # noqa: BLE001
            err.append(exc)
            return -1

    from ._lib import ALLREDUCE_CB, GATHER_CB

    cb_ar, cb_g = ALLREDUCE_CB(allreduce), GATHER_CB(gather)
    alphas, betas = np.zeros(k), np.zeros(k)
    beta_last, steps = ctypes.c_double(), ctypes.c_int()
    pd = ctypes.POINTER(ctypes.c_double)
    h_rows = ctypes.c_void_p(op.row_ptr(part.r0, nl) if nl else op.tensor.data_ptr())
    status = lib().chfsi_lanczos_rows_z(ctx(), n, k, h_rows, op.ld, op.conj, part.r0, nl,
                                        dptr(q0d), dptr(basis), dptr(ws), cb_ar, cb_g, None,
                                        alphas.ctypes.data_as(pd), betas.ctypes.data_as(pd),
                                        ctypes.byref(beta_last), ctypes.byref(steps))
    if err:
        raise err[0]
    check(status, "lanczos (row-sharded)")
    return alphas, betas, beta_last.value, steps.value


# ----------------------------------------------- row-sharded reduction ---

class RowOperator(Operator):
    """One rank's row block of the Hermitian operator H = L^-1 A L^-H:
    rows [row0, row0 + rows) stored as the COLUMN block H[:, row0:row0+rows]
    (column-major, ld n) — by Hermitian symmetry column r read with the
    conj flag is row r, so K1 and the row-sharded Lanczos read their rows in
    place (`Operator.row_ptr`). No rank holds the rest of H."""

    __slots__ = ()

    def __init__(self, block, n, row0):  # noqa: super().__init__ would want a square matrix
        if block.dim() != 2 or block.shape[0] != n or (block.shape[1] > 1 and block.stride(0) != 1):
            raise ValueError("row block must be a column-major n x rows tensor")
        self.tensor, self.n, self.row0, self.rows = block, n, row0, block.shape[1]
        self.ld = max(int(block.stride(1)), n) if self.rows > 1 else n
        self.conj = 1


class DeviceLinalg:
    """Local dense kernels of the sharded reduction: cuSOLVER potrf and
    cuBLAS ZTRSM through libchfsi (tests inject a host restatement)."""

    @staticmethod
    def potrf(b):
        """Lower Cholesky factor (column-major device block, upper zeroed) of
        the Hermitian ``b``; NotPositiveDefiniteError when b is not HPD."""
        import ctypes

        from ._device import to_fblock

        l = to_fblock(b, copy=True)
        info = ctypes.c_int()
        check(lib().chfsi_potrf_z(ctx(), l.shape[0], dptr(l), l.stride(1), ctypes.byref(info)),
              "cholesky (sharded reduction)")
        return l

    @staticmethod
    def trsm(l, x, conj_transpose=False):
        """x <- L^-1 x (or L^-H x) in place, x a column-major n x k block."""
        check(lib().chfsi_trsm_z(ctx(), b"L", b"C" if conj_transpose else b"N", x.shape[0],
                                 x.shape[1], dptr(l), l.stride(1), dptr(x), max(x.stride(1),
                                                                                 x.shape[0])),
              "triangular solve (sharded reduction)")
        return x


def _fcols(n, k, like):
    return torch.empty((k, n), dtype=torch.complex128, device=like.device).t()


def _block_transpose(comm, cols):
    """T = (H[cols_p, :])^H from the column blocks H[:, cols_q] of all ranks:
    rank q sends the rows cols_p of its block to rank p (one all-to-all of
    kblk x kblk tiles); T[cols_q, :] = (block_q[cols_p, :])^H."""
    part = comm.part
    n, kb, P = part.n, part.kblk, part.world
    send = torch.zeros((P, kb, kb), dtype=torch.complex128, device=cols.device)
    for q in range(P):
        q0, qr = part.block_range(q)
        if qr and part.rows:  # rows of destination q's column range, this rank's columns
            send[q, :part.rows, :qr] = cols[q0:q0 + qr, :].t()  # [my col][their row]
    recv = comm.alltoall_blocks(send)  # recv[q][q's col][my row] = H[my rows, q's cols]^T
    out = _fcols(n, part.rows, cols)
    for q in range(P):
        q0, qr = part.block_range(q)
        if qr and part.rows:
            # (H[cols_p, cols_q])^H as a column-major (qr x rows) block: element
            # [i, j] = conj(H[p0 + j, q0 + i]) = conj(recv[q][i, j])
            out[q0:q0 + qr, :] = recv[q, :qr, :part.rows].conj()
    return out


def to_standard_rows(a, b, comm, linalg=DeviceLinalg):
    """Row-sharded reduction to standard form (reference reduction.py:102-113
    split over the ranks of ``comm``): every rank gets ITS row block of
    H = L^-1 A L^-H (as a RowOperator) and the Cholesky factor L.

    * L = chol(B) on every rank (n^3/3 complex MACs, replicated: the
      factor is needed whole by both solves and the back-transform);
    * Z_p = L^-1 A[:, cols_p] — this rank's column block (TRSM, n^2 kblk);
    * W_p = (Z[cols_p, :])^H by one all-to-all of kblk x kblk tiles;
    * H[:, cols_p] = L^-1 W_p (TRSM), since H = L^-1 Z^H;
    * symmetrised (h + h^H)/2 as the reference does, the transpose part
      through a second all-to-all.
    The O(n^3) triangular solves are split P ways; no rank ever holds the
    rest of H. ``a``/``b``: full Hermitian matrices (numpy or torch, any
    layout) on every rank."""
    from ._device import to_device_matrix

    part = comm.part
    n = part.n
    dev_b = to_device_matrix(b) if linalg is DeviceLinalg else b
    l = linalg.potrf(dev_b)
    a_d = to_device_matrix(a) if linalg is DeviceLinalg else a
    r0, rows = part.r0, part.rows
    z = _fcols(n, rows, l)
    if rows:
        z.copy_(a_d[:, r0:r0 + rows])
        linalg.trsm(l, z)
    w = _block_transpose(comm, z)  # (Z[cols_p, :])^H
    del z
    if rows:
        linalg.trsm(l, w)  # H[:, cols_p]
    t = _block_transpose(comm, w)  # (H[cols_p, :])^H
    w.add_(t).mul_(0.5)
    return RowOperator(w, n, r0), l


def back_transform_rows(l, y, comm, linalg=DeviceLinalg):
    """x = L^-H y (reduction.py:122-134) with the columns of the full
    standard-form block ``y`` (n x k, the same on every rank) split over
    the ranks; every rank returns the full x."""
    part = comm.part
    n, k = y.shape
    P = part.world
    cb = -(-k // P) if k else 0
    c0, c1 = min(k, part.rank * cb), min(k, (part.rank + 1) * cb)
    mine = torch.zeros((cb, n), dtype=torch.complex128, device=y.device)  # [col][row]
    if c1 > c0:
        blk = _fcols(n, c1 - c0, y)
        blk.copy_(y[:, c0:c1])
        linalg.trsm(l, blk, conj_transpose=True)
        mine[: c1 - c0].copy_(blk.t())
    every = comm.allgather_blocks(mine)  # [P][cb][n]
    out = torch.empty((k, n), dtype=torch.complex128, device=y.device)
    for q in range(P):
        q0, q1 = min(k, q * cb), min(k, (q + 1) * cb)
        if q1 > q0:
            out[q0:q1].copy_(every[q, : q1 - q0])
    return out.t()
