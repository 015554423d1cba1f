"""Sequence drivers on the device — drop-in for `spectral_chain.harness`
(reference `harness.py:149-336`).

`run_experiment(spec)` is the reference's four-stage warm-start experiment
(dense oracle of problem l-1 -> random-start and warm-start ChFSI cells of
problem l -> oracle check -> report rows), `emit_report` its CSV/JSON
writer. `solve_sequence` (additive) is the production driver with two
protocols over a correlated sequence of pencils (label 1..N):

* ``mode="harness"`` — the reference's parity protocol (harness.py:235-255):
  problem l >= 2 is warm-started from the DENSE eigendecomposition of
  problem l-1 (here cuSOLVER zheevd on the device), lambda_1 and
  lambda_{blk+1} taken from that full spectrum; rng ``(seed, l, 1)``.
* ``mode="chained"`` — production warm starts: problem l >= 2
  starts from the previous ChFSI tail block ``[locked | unlocked panel]``
  and its Ritz window; no dense solve anywhere.

Problem 1 is always a cold start with rng ``(seed, 1, 0)``. Every problem
runs to_standard -> chfsi_solve -> back_transform on the device.
"""

from __future__ import annotations

import csv
import gc
import itertools
import json
import os
import statistics
import time
from concurrent.futures import Future, ThreadPoolExecutor, wait
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np
import torch

from ._device import array_output, to_device_matrix
from .chfsi import ChfsiConfig, ChfsiGuess, PrefetchedStart, WarmLanczos, chfsi_solve, warm_lanczos
from .linalg import hermitian_eig
from .reduction import EigenPencil, EigenSolution, back_transform, stage_standard, to_standard

__all__ = [
    "GenerateSource",
    "LoadSource",
    "BaselineSource",
    "ExperimentSpec",
    "ExperimentRow",
    "ExperimentReport",
    "OracleMismatchError",
    "SOLVERS",
    "REPORT_FIELDS",
    "oracle_solve",
    "run_experiment",
    "emit_report",
    "replace_tracked",
    "ProblemResult",
    "solve_sequence",
    "check_oracle",
]

_ORACLE_TOL = 1e-8  # harness.py:49


class OracleMismatchError(RuntimeError):
    """An iterative solve disagreed with the direct solver (harness.py:68-69)."""


def oracle_solve(pencil, nev):
    """Dense direct solution of a pencil on the device (harness.py:149-161):
    (standard-form solution of ``nev`` pairs, reduced problem, full spectrum)."""
    sp = to_standard(pencil)
    values, vectors = hermitian_eig(sp.h)
    sol = EigenSolution(values=values[:nev], vectors=vectors[:, :nev], form="standard",
                        label=pencil.label)
    return sol, sp, values


def check_oracle(values, oracle_values, label, start="warm"):
    """|lambda - lambda_dense| <= 1e-8 * spectrum scale (harness.py:179-185)."""
    scale = float(max(abs(oracle_values[0]), abs(oracle_values[-1]), 1e-300))
    err = float(np.abs(np.asarray(values) - oracle_values[: len(values)]).max(initial=0.0))
    if err > _ORACLE_TOL * scale:
        raise OracleMismatchError(
            f"problem {label} ({start} start): eigenvalue error {err:.3e} exceeds "
            f"{_ORACLE_TOL:.0e} on spectrum scale {scale:.3e}")
    return err


@dataclass
class ProblemResult:
    label: int
    values: np.ndarray
    solution: EigenSolution          # generalized form (x = L^-H y), device vectors
    standard_vectors: object         # standard-form y (device) — for parity checks
    report: object
    t_reduce: float = 0.0
    t_solve: float = 0.0
    t_back: float = 0.0
    dense_values: np.ndarray | None = None
    extra: dict = field(default_factory=dict)


def _as_pencil(p):
    if isinstance(p, EigenPencil):
        return p
    label, a, b = p
    return EigenPencil(a=a, b=b, label=label)


_SIDE_STREAMS = {}


def side_stream(device=None):
    """One persistent side stream per device (and so one libchfsi context for
    it): creating a stream per call would create a context per call."""
    dev = torch.cuda.current_device() if device is None else device
    st = _SIDE_STREAMS.get(dev)
    if st is None:
        st = _SIDE_STREAMS[dev] = torch.cuda.Stream(device=dev)
    return st


_SIDE_WORKERS = {}
_BACK_SIDE_MAX_N = 8192  # side-stream back-transform up to this n (memory, see solve_sequence)


def side_worker(device):
    """One persistent worker thread per device that issues the side stream's
    work (its libchfsi contexts are per thread, so a thread per call would
    build new cuBLAS/cuSOLVER handles per call)."""
    w = _SIDE_WORKERS.get(device)
    if w is None:
        w = _SIDE_WORKERS[device] = ThreadPoolExecutor(max_workers=1,
                                                       thread_name_prefix="chfsi-side")
    return w


class _StagingSlots:
    """Two preallocated (H, L) buffer pairs that stage_standard writes into
    in turn (n > _BACK_SIDE_MAX_N). Problem l+2 reuses problem l's pair: its
    staging is issued after problem l's solve and back-transform finished
    (the main-stream synchronisation at the end of every problem), so at
    most two H/L pairs ever exist and no n x n block goes through the
    caching allocator per problem — at C5 each pair is 12.8 GB, and
    per-stream allocator pools otherwise left freed pairs unusable by the
    next staging (OOM with the default bench warm-ups)."""

    def __init__(self, n, device, count=2):
        self.pairs = [(torch.empty((n, n), dtype=torch.complex128, device=device),
                       torch.empty((n, n), dtype=torch.complex128, device=device))
                      for _ in range(count)]
        self.k = 0

    def take(self, side):
        pair = self.pairs[self.k]
        self.k = (self.k + 1) % len(self.pairs)
        for t in pair:
            t.record_stream(side)
        return pair


# the staging pairs of small sequences, reused by later calls on the same
# stream: problem l+2's staging is ordered after problem l's solve (the event
# it waits on) and back-transform (same side stream), and a later call's
# first staging after everything of the previous call
_SLOT_CACHE = {}


def _item_n(item):
    a = item.a if isinstance(item, EigenPencil) else item[1]
    return int(a.shape[0])


def _stage(item, side, ready=None, slot=None, warm_seed=None):
    """Upload, validate and reduce one pencil on the side stream without any
    host synchronisation (the validation results land in page-locked memory
    and are checked when the problem is about to be solved, raising the
    reference's exceptions then); returns (pencil, StandardProblem, ready
    event, pending checks).

    ``ready`` is an event recorded on the caller's stream right after the
    item was produced: a lazy device generator queues the work that writes
    A and B on that stream inside ``next()``, so the side stream must wait
    for it before reading them.

    ``warm_seed`` (worker thread only: it blocks until the side stream gets
    there): also run the problem's warm-start Lanczos bound estimate on the
    side stream right behind its reduction — it needs only H, not the
    previous solve — so the solve starts its filter at once instead of
    spending ~0.6 ms of host round trips (q0 upload, 10 Lanczos steps, the
    tridiagonal eigenvalues on the host) with the main stream idle."""
    with torch.cuda.stream(side):
        if ready is not None:
            side.wait_event(ready)
        a_b = (item.a, item.b) if isinstance(item, EigenPencil) else tuple(item[1:3])
        for t in a_b:  # allocated on another stream, read on this one
            if isinstance(t, torch.Tensor) and t.is_cuda:
                t.record_stream(side)
        if isinstance(item, EigenPencil):  # validated at construction
            pencil, sp, checks = stage_standard(item.a, item.b, item.label, check_hermitian=False,
                                                out=slot)
        else:
            label, a, b = item
            pencil, sp, checks = stage_standard(a, b, label, out=slot)
        ev = torch.cuda.Event()
        ev.record(side)
        warm = warm_lanczos(sp.h, warm_seed) if warm_seed is not None else None
    return pencil, sp, ev, checks, warm


class _OutputArena:
    """One device block per sequence call holding every problem's outputs —
    the chained tail (n x blk) and the eigenvector block (n x nev) — carved
    as column-major views. One allocation of the same size per call reuses
    the same cached segment of torch's allocator (the previous call's results
    released it), where per-problem allocations and the round-1 "reserve and
    free" trick made the allocator cudaMalloc new segments at arbitrary
    points (measured: +25-90 ms in ~1 of 5 C2 sequences, in the reservation
    or inside a solve). The views keep the block alive as long as any result
    is alive."""

    def __init__(self, count, n, blk, nev, device):
        self.per = n * (blk + nev)
        self.buf = torch.empty(count * self.per, dtype=torch.complex128, device=device)
        self.k = 0
        self.count = count

    def take(self, n, blk, nev):
        if self.k >= self.count or n * (blk + nev) != self.per:
            return None
        base = self.buf[self.k * self.per:(self.k + 1) * self.per]
        self.k += 1
        tail = base[: n * blk].view(blk, n).t()
        vecs = base[n * blk:].view(nev, n).t()
        return tail, vecs


def _output_arena(pencil, cfg, pencils):
    """The per-call output arena (None when the sequence length is unknown
    or the outputs would take more than 5 % of the device memory)."""
    try:
        length = len(pencils)
    except TypeError:
        return None
    n = pencil.n
    blk = cfg.resolve(n)[0]
    dev = torch.cuda.current_device()
    total = _TOTAL_MEM.get(dev)
    if total is None:
        total = _TOTAL_MEM[dev] = torch.cuda.get_device_properties(dev).total_memory
    if length * n * (blk + cfg.nev) * 16 > total // 20:
        return None
    # An arena of this shape is reused when none of its results is alive any
    # more (the storage is referenced by the cached tensor alone): no
    # allocation at all in a steady sequence of calls. Up to three are kept
    # per shape, so a caller that still holds the previous call's results
    # while it starts the next one (or whose results sit in not-yet-collected
    # reference cycles) alternates between cached blocks instead of making
    # the allocator cudaMalloc a new segment every other call (measured on
    # these boxes: 25-135 ms of host stall per cudaMalloc, 2 of 10 C2 steps).
    key = (dev, torch.cuda.current_stream().cuda_stream, length, n, blk, cfg.nev)
    pool = _ARENAS.setdefault(key, [])
    for cached in pool:
        if _storage_users(cached.buf) <= 1:
            cached.k = 0
            return cached
    arena = _OutputArena(length, n, blk, cfg.nev, dev)
    pool.append(arena)
    if len(pool) > 3:  # every cached block is in use: forget the oldest
        pool.pop(0)
    if len(_ARENAS) > 4:  # a few shapes at most
        _ARENAS.pop(next(iter(_ARENAS)))
    return arena


def _storage_users(t):
    """Tensors (the base and its views) sharing ``t``'s storage."""
    return torch._C._storage_Use_Count(t.untyped_storage()._cdata) - 1


_ARENAS = {}
_TOTAL_MEM = {}


def solve_sequence(pencils, cfg, seed=0, mode="chained", keep_standard=False, on_problem=None,
                   overlap=True, shard=None):
    """Solve a correlated sequence on the device.

    ``pencils`` yields EigenPencil or ``(label, A, B)`` (numpy or torch).
    ``cfg`` is a ChfsiConfig (``nex`` accepted). Returns a list of
    ProblemResult; ``on_problem(result)`` is called after each problem.

    With ``overlap`` the upload + reduction to standard form of problem l+1
    runs on a side stream while problem l is being solved (the reduction
    does not depend on the previous solve), hiding it behind the solver's
    latency-bound phases; the back-transform of problem l runs on the same
    side stream behind problem l+1's solve (``CHFSI_BACK_ON_SIDE=0`` keeps
    it on the caller's stream). Results are identical either way.

    ``shard`` (multi-GPU, one process per GPU, every rank calling with the
    same pencils): True, a process group or a `distributed.RowComm` runs
    the row-sharded path — per problem the reduction leaves each rank only
    its row block of H (`distributed.to_standard_rows`), the solve is
    row-sharded (`chfsi_solve(shard=...)`) and the back-transform splits the
    eigenvector columns over the ranks; every rank returns the full results
    (chained mode; the harness protocol needs the dense spectrum of the
    whole H and is not sharded).
    """
    if mode not in ("chained", "harness"):
        raise ValueError(f"unknown mode {mode!r}")
    if shard is not None and shard is not False:
        if mode != "chained":
            raise NotImplementedError("the row-sharded sequence runs mode='chained' (the harness "
                                      "protocol needs the dense eigendecomposition of the whole H)")
        return _solve_sequence_sharded(pencils, cfg, seed, keep_standard, on_problem, shard)
    caller = torch.cuda.current_stream()
    it = iter(pencils)
    first = next(it, None)
    if first is None:
        return []
    # (a list keeps its length for the output reservation; other iterables
    # go on lazily behind the peeked first item)
    seq = pencils if isinstance(pencils, (list, tuple)) else itertools.chain([first], it)
    # (also without the side stream: the solver's library handles then keep
    # one history across driver modes — cuBLAS's algorithm choices depend on
    # it, and results would differ in the last bit between modes). Large n:
    # the staged reduction of problem l+1 (~0.5 s at n = 12000) needs real SM
    # time beside the solve, so the solver stream keeps the side stream's
    # priority there (C4: a high-priority solver starved it, +2 s of waits).
    high = _item_n(first) <= _BACK_SIDE_MAX_N
    solver = solver_stream(high=high) if _PRIORITY else caller
    if solver is caller:
        return _solve_sequence_on(seq, cfg, seed, mode, keep_standard, on_problem, overlap)
    # The solver's own work runs on a HIGH-priority stream: the block
    # scheduler then places its CTAs first whenever SMs free up, so the
    # side stream's reduction of problem l+1 fills the solver's latency gaps
    # instead of holding SMs that the solver's short, serial kernels
    # (potrf, TRSM, the w x w eigensolver) are waiting for.
    solver.wait_stream(caller)
    with torch.cuda.stream(solver):
        out = _solve_sequence_on(seq, cfg, seed, mode, keep_standard, on_problem, overlap)
    caller.wait_stream(solver)
    for r in out:  # results were allocated on the solver stream, used on the caller's
        for t in (r.solution.vectors if r.solution is not None else None, r.standard_vectors,
                  r.report.tail_vectors):
            if isinstance(t, torch.Tensor) and t.is_cuda:
                t.record_stream(caller)
    return out


_PRIORITY = os.environ.get("CHFSI_STREAM_PRIORITY", "1") != "0"
# CHFSI_WARM_AHEAD=0: the warm-start Lanczos estimate inside the solve (A/B)
_WARM_AHEAD = os.environ.get("CHFSI_WARM_AHEAD", "1") != "0"
# CHFSI_STAGE_DEPTH=1: stage only problem l+1 during solve l (two H/L pairs; A/B)
_STAGE_DEPTH = int(os.environ.get("CHFSI_STAGE_DEPTH", "2"))
# CHFSI_DRIVER_TRACE=1: (event, perf_counter) marks of the driver's host
# timeline appended to DRIVER_TRACE (diagnostics: tools/diag/step_outliers.py)
_TRACE_ON = os.environ.get("CHFSI_DRIVER_TRACE") == "1"
DRIVER_TRACE = []


def _mark(what):
    if _TRACE_ON:
        DRIVER_TRACE.append((what, time.perf_counter()))
_SOLVER_STREAMS = {}


def solver_stream(device=None, high=True):
    """One persistent solver stream per device and priority class: highest
    priority (small n) or the default priority of the side stream (large n)."""
    dev = torch.cuda.current_device() if device is None else device
    st = _SOLVER_STREAMS.get((dev, high))
    if st is None:
        st = _SOLVER_STREAMS[(dev, high)] = torch.cuda.Stream(device=dev,
                                                              priority=-100 if high else 0)
    return st


def _solve_sequence_on(pencils, cfg, seed, mode, keep_standard, on_problem, overlap):
    """solve_sequence's single-GPU body on the current stream."""
    _mark("enter")
    out = []
    guess = None
    main = torch.cuda.current_stream()
    side = side_stream() if overlap else main
    back_side = side is not main and os.environ.get("CHFSI_BACK_ON_SIDE", "1") != "0"

    def produced():
        # every input is handed to the side stream behind an event recorded
        # on the caller's stream AFTER the iterator produced it (device work
        # a lazy generator queues inside next() is then visible to the side)
        if side is main:
            return None
        ev = torch.cuda.Event()
        ev.record(main)
        return ev

    it = iter(pencils)
    first = next(it, None)
    slots = None
    # Side-stream work (staging of problems l+1.., back-transform of problem
    # l) is ISSUED by one worker thread: its host-side launch cost (~1 ms per
    # problem) then overlaps the solve instead of leaving the main stream
    # idle between problems (the native loop runs without the GIL). The
    # worker's FIFO keeps the side stream's order: stage(l+2), back(l), ...
    # (large n: seconds per problem make the worker's ~1 ms moot, and issuing
    # inline keeps the allocator's frees ordered as at C5's memory limit)
    threaded = (side is not main and os.environ.get("CHFSI_SIDE_WORKER", "1") != "0"
                and (first is None or _item_n(first) <= _BACK_SIDE_MAX_N))
    # Staging depth: with the worker, problems l+1 AND l+2 are staged while l
    # is solved (three H/L pairs in rotation). The side stream only gets the
    # SM time the high-priority solver leaves, so a reduction handed over at
    # the start of solve l finishes near its end — the short late solves of a
    # sequence then waited 0.7-1.2 ms each for their operator, and anything
    # queued behind the reduction (the warm-start Lanczos estimate) landed on
    # the critical path. One problem further ahead, both are long done.
    depth = 2 if threaded and _STAGE_DEPTH >= 2 else 1
    if first is not None:
        n0 = _item_n(first)
        if n0 > _BACK_SIDE_MAX_N:  # per call: 12.8 GB per pair at C5
            slots = _StagingSlots(n0, torch.cuda.current_device())
        else:  # kept across calls: no per-problem 2 n^2 allocations at all
            key = (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream, n0, depth + 1)
            slots = _SLOT_CACHE.get(key)
            if slots is None:
                if len(_SLOT_CACHE) >= 2:
                    _SLOT_CACHE.pop(next(iter(_SLOT_CACHE)))
                slots = _SLOT_CACHE[key] = _StagingSlots(n0, torch.cuda.current_device(), depth + 1)

    def slot():
        return None if slots is None else slots.take(side)

    staged = _stage(first, side, produced(), slot()) if first is not None else None
    _mark("first stage issued")
    prefetch = None
    arena = None
    if staged is not None:
        arena = _output_arena(staged[0], cfg, pencils)
        _mark("output arena")
        # problem 1 is a cold start: its draws (q0, then the n x blk block)
        # run on a host thread from here on, behind its upload and reduction
        p0 = staged[0]
        prefetch = PrefetchedStart(np.random.default_rng((seed, p0.label, 0)), p0.n,
                                   cfg.resolve(p0.n)[0])
    dev = torch.cuda.current_device()
    worker = side_worker(dev) if threaded else None
    issued = []
    # Side-stream jobs are collected here and handed to the worker only once
    # the next solve has queued its first device work and entered the native
    # loop (chfsi_solve's `_hooks`): the worker's Python then runs while the
    # main thread is inside the GIL-free loop, instead of competing for the
    # GIL with the main thread's between-problem bookkeeping and the next
    # problem's set-up (measured: ~0.5 ms of device idle per C2 problem).
    deferred = []

    class _Later:
        def __init__(self, fn, args):
            self.fn, self.args, self.fut = fn, args, None

        def result(self):
            if self.fut is None:
                flush()
            return self.fut.result()

    def flush():
        jobs = list(deferred)
        deferred.clear()
        for job in jobs:
            job.fut = submit(job.fn, *job.args)

    def later(fn, *args):
        if worker is None:
            return submit(fn, *args)
        job = _Later(fn, args)
        deferred.append(job)
        return job

    def on_device(fn, *args):
        with torch.cuda.device(dev):
            return fn(*args)

    def submit(fn, *args):
        if worker is None:  # CHFSI_SIDE_WORKER=0: issued inline, same stream order
            fut = Future()
            fut.set_result(fn(*args))
            return fut
        fut = worker.submit(on_device, fn, *args)
        issued.append(fut)
        return fut

    def back_on_side(solved, l_factor, sol):
        # x = L^-H y of problem l on the side stream, behind its solve: it
        # overlaps problem l+1's solve (the chained guess is the standard-form
        # tail, not x); the caller's stream joins at the end.
        with torch.cuda.stream(side):
            side.wait_event(solved)
            gsol = back_transform(l_factor, sol, inplace=not keep_standard)
            done = torch.cuda.Event()
            done.record(side)
        l_factor.record_stream(side)
        gsol.vectors.record_stream(side)
        return gsol, done

    pending = []  # (result, future of the side-stream back-transform)
    # No cyclic GC passes inside the sequence: a full collection of a
    # torch-sized heap holds the GIL for 50-400 ms, and whichever thread
    # triggers it stalls the other's return from the native loop (measured
    # with the side worker: problem 9 of C2 sequences +15..360 ms in 5 of
    # 24 steps; none in 24 steps without collections). Cycles are collected
    # as usual once the call returns.
    gc_on = gc.isenabled()
    gc.disable()

    def settle(res, fut):
        res.solution, done = fut.result()
        return done

    _mark("first staged")
    queue = [staged] if staged is not None else []  # staged problems, in order (at most `depth` ahead)
    exhausted = False
    try:
        while queue:
            _mark("problem top")
            t0 = time.perf_counter()
            staged = queue.pop(0)
            if not isinstance(staged, tuple):  # issued by the worker during an earlier solve
                fut, staged = staged, staged.result()
                fut = getattr(fut, "fut", fut)
                if fut in issued:  # a done future holds its result: drop it, or every
                    issued.remove(fut)  # problem's H and L would live until the call ends
            pencil, sp, ev, checks, warm = staged
            ev.synchronize()  # long done for l >= 2: staged while an earlier problem was solved
            checks.raise_if_invalid()
            main.wait_event(ev)
            if side is not main:
                for t in (sp.h, sp.cholesky_factor, pencil.a, pencil.b):
                    t.record_stream(main)
            t1 = time.perf_counter()
            while len(queue) < depth and not exhausted:
                nxt = next(it, None)
                if nxt is None:
                    exhausted = True
                elif slots is not None and _item_n(nxt) != slots.pairs[0][0].shape[0]:
                    raise ValueError("all pencils of a sequence must share one dimension")
                elif side is not main:
                    # (with the worker thread the problem's warm-start Lanczos
                    # estimate runs ahead too; its seed is the warm start's)
                    nlab = nxt.label if isinstance(nxt, EigenPencil) else nxt[0]
                    wseed = (seed, nlab, 1) if worker is not None and _WARM_AHEAD else None
                    queue.append(later(_stage, nxt, side, produced(), slot(), wseed))
                else:
                    queue.append(_stage(nxt, side, None, slot()))
            t_stage = time.perf_counter() - t1
            t1 = time.perf_counter()
            n = pencil.n
            blk = cfg.resolve(n)[0]
            if mode == "harness" and blk >= n:
                raise ValueError(f"chfsi warm starts need blk < n (blk={blk}, n={n})")
            start = 0 if guess is None else 1
            if guess is None or warm is None:
                warm = None  # (cold restart: the estimate drawn for a warm start is not used)
            if prefetch is not None:  # (always problem 1: guess is None there)
                rng, prefetch = prefetch, None
            elif warm is not None:
                rng = warm.rng  # the warm start's generator, already past the q0 draw
            else:
                rng = np.random.default_rng((seed, pencil.label, start))
            _mark("solve start")
            out_bufs = arena.take(n, blk, cfg.nev) if arena is not None else None
            sol, rep = chfsi_solve(sp.h, cfg, guess=guess, rng=rng, label=pencil.label,
                                   _hooks=flush if deferred else None, _sync=False, _out=out_bufs,
                                   _warm=warm)
            _mark("solve end")
            t2 = time.perf_counter()
            back = None
            # at large n the side-stream back-transform would keep L of problem
            # l (6.4 GB at C5) alive next to the staged l+1: run it inline there
            if back_side and n <= _BACK_SIDE_MAX_N:
                solved = torch.cuda.Event()
                solved.record(main)
                back = later(back_on_side, solved, sp.cholesky_factor, sol)
                gsol = None  # filled from `back`
            else:
                gsol = back_transform(sp.cholesky_factor, sol, inplace=not keep_standard)
            # no host synchronisation here: the next problem's set-up overlaps
            # this one's last device work (slot reuse at large n is ordered by
            # the `produced` event the next staging waits on)
            t3 = time.perf_counter()
            res = ProblemResult(label=pencil.label, values=sol.values, solution=gsol,
                                standard_vectors=sol.vectors if keep_standard else None,
                                report=rep, t_reduce=t1 - t0 - t_stage, t_solve=t2 - t1,
                                t_back=t3 - t2)
            res.extra["t_stage_next"] = t_stage
            if mode == "harness":
                dv, dvec = hermitian_eig(sp.h)
                res.dense_values = dv
                guess = ChfsiGuess(vectors=dvec[:, :blk], lambda1=float(dv[0]),
                                   lambda_blk_plus_1=float(dv[blk]))
            else:
                if rep.tail_vectors is not None and rep.tail_vectors.shape[1] == blk and sol.nev:
                    guess = ChfsiGuess(vectors=rep.tail_vectors, lambda1=float(sol.values[0]),
                                       lambda_blk_plus_1=float(rep.lambda_blk_plus_1))
                else:  # a partial solve leaves no full block: restart cold
                    guess = None
            out.append(res)
            if back is not None:
                pending.append((res, back))
            if on_problem is not None:
                if back is not None:
                    settle(res, back).synchronize()
                on_problem(res)
            del sp
    finally:
        _mark("loop end")
        flush()
        wait(issued)  # nothing the worker issues outlives this call
        _mark("worker idle")
        if gc_on:
            gc.enable()
    try:
        for res, fut in pending:
            settle(res, fut)  # re-raises a failed back-transform
    finally:
        # the closures above sit in reference cycles (collected only by a
        # later cyclic GC pass): empty the lists they hold, or the futures in
        # them would keep every result's output block alive past the caller's
        # last reference, and the next call could not reuse it
        pending.clear()
        issued.clear()
        deferred.clear()
    main.wait_stream(side)
    _mark("exit")
    return out


def _row_comm(shard, n):
    """A RowComm (or a stand-in with the same interface) for ``shard``."""
    if hasattr(shard, "part") and hasattr(shard, "allreduce_"):
        if shard.part.n != n:
            raise ValueError(f"communicator is for n={shard.part.n}, the pencils have n={n}")
        return shard
    from .distributed import RowComm

    group = shard if not isinstance(shard, (bool, int)) else None
    chunks = shard if isinstance(shard, int) and not isinstance(shard, bool) else 2
    return RowComm(n, group=group, chunks=chunks)


def _solve_sequence_sharded(pencils, cfg, seed, keep_standard, on_problem, shard):
    """solve_sequence over row-sharded operators (see its docstring), chained
    warm starts. No side stream: the reduction's all-to-alls and the solve's
    collectives stay in one stream order on every rank."""
    from .distributed import back_transform_rows, to_standard_rows

    out, guess, comm = [], None, None
    for item in pencils:
        pencil = _as_pencil(item)
        n = pencil.n
        if comm is None:
            comm = _row_comm(shard, n)
        elif comm.part.n != n:
            raise ValueError("all pencils of a sequence must share one dimension")
        blk = cfg.resolve(n)[0]
        t0 = time.perf_counter()
        op, l_factor = to_standard_rows(pencil.a, pencil.b, comm)
        t1 = time.perf_counter()
        rng = np.random.default_rng((seed, pencil.label, 0 if guess is None else 1))
        sol, rep = chfsi_solve(op, cfg, guess=guess, rng=rng, label=pencil.label, shard=comm)
        t2 = time.perf_counter()
        x = back_transform_rows(l_factor, sol.vectors, comm)
        gsol = replace(sol, vectors=x, form="generalized")
        torch.cuda.current_stream().synchronize()
        t3 = time.perf_counter()
        res = ProblemResult(label=pencil.label, values=sol.values, solution=gsol,
                            standard_vectors=sol.vectors if keep_standard else None, report=rep,
                            t_reduce=t1 - t0, t_solve=t2 - t1, t_back=t3 - t2)
        if rep.tail_vectors is not None and rep.tail_vectors.shape[1] == blk and sol.nev:
            guess = ChfsiGuess(vectors=rep.tail_vectors, lambda1=float(sol.values[0]),
                               lambda_blk_plus_1=float(rep.lambda_blk_plus_1))
        else:  # a partial solve leaves no full block: restart cold
            guess = None
        out.append(res)
        if on_problem is not None:
            on_problem(res)
        del op, l_factor
    return out


def default_config(cfg):
    """ChfsiConfig for a BASELINE config (sequence.BaselineConfig)."""
    return ChfsiConfig(nev=cfg.nev, nex=cfg.nex, deg=cfg.deg, tol=cfg.tol,
                       adaptive_degree=cfg.adaptive_degree)


# ------------------------------------------------ the experiment protocol ---
# run_experiment(spec) -> ExperimentReport: the reference's four-stage
# warm-start experiment (harness.py:188-289) with every solve on the device.

# The reference's solver names (harness.py:45); only ChFSI is the hot path
# this package rebuilds, the LOBPCG baselines stay in the reference.
SOLVERS = ("chfsi", "lobpcg", "lobpcg-generalized")
_OUT_OF_SCOPE = ("lobpcg", "lobpcg-generalized")

REPORT_FIELDS = [  # CSV schema (harness.py:52-65); JSON rows carry the same keys
    "ell", "t_random_s", "t_approx_s", "speedup_time", "matvecs_random", "matvecs_approx",
    "speedup_matvec", "filtered_random", "filtered_approx", "inner_loops_random",
    "inner_loops_approx", "median_angle",
]


@dataclass
class GenerateSource:
    """Generate with the reference's generator (harness.py:72-78)."""

    n: int
    schedule: object  # sequence.CorrelationSchedule
    seed: int = 0


@dataclass
class LoadSource:
    """A saved sequence directory: npy or the reference's Matrix Market
    files (harness.py:81-85)."""

    directory: str


@dataclass
class BaselineSource:
    """Additive: the BASELINE.json generator (`sequence.iter_baseline_sequence`),
    computed on the device when ``device`` is true."""

    n: int
    length: int
    seed: int = 0
    device: bool = True


@dataclass
class ExperimentSpec:
    """harness.py:88-107 — same fields, defaults and validation."""

    source: object
    solver: str
    nev: int
    solver_overrides: dict = field(default_factory=dict)
    tracked_fraction: float = 1.0
    repetitions: int = 5
    seed: int = 0

    def __post_init__(self):
        if self.solver not in SOLVERS:
            raise ValueError(f"unknown solver {self.solver!r}, expected one of {SOLVERS}")
        if self.repetitions < 1:
            raise ValueError("repetitions must be >= 1")
        if not 0 < self.tracked_fraction <= 1:
            raise ValueError("tracked_fraction must be in (0, 1]")
        if self.nev < 1:
            raise ValueError("nev must be >= 1")


@dataclass
class ExperimentRow:
    """One compared problem, labels 2..N (harness.py:110-129)."""

    ell: int
    t_random_s: float
    t_approx_s: float
    speedup_time: float
    matvecs_random: int
    matvecs_approx: int
    speedup_matvec: float
    filtered_random: int
    filtered_approx: int
    inner_loops_random: int
    inner_loops_approx: int
    median_angle: float
    max_residual_random: float
    max_residual_approx: float
    converged_random: bool
    converged_approx: bool


@dataclass
class ExperimentReport:
    """harness.py:132-146."""

    rows: list
    n: int
    length: int
    solver: str
    nev: int
    blk: int
    repetitions: int
    tracked_fraction: float
    seed: int
    warnings: list = field(default_factory=list)

    @property
    def all_converged(self):
        return all(r.converged_random and r.converged_approx for r in self.rows)


def replace_tracked(sol, count):
    """The lowest ``count`` pairs of a solution (harness.py:292-295)."""
    count = min(count, sol.nev)
    return replace(sol, values=sol.values[:count], vectors=sol.vectors[:, :count])


def _source_pencils(source):
    """(n, length, lazy iterator of device EigenPencils) of a spec source."""
    from . import pencil_io
    from .sequence import iter_baseline_sequence, iter_generated_sequence

    def device_pencils(items):
        for lab, a, b in items:
            # (memory-mapped files are read-only: np.require copies those)
            yield EigenPencil(a=to_device_matrix(np.require(a, requirements=["C", "W"]))
                              if not isinstance(a, torch.Tensor) else a,
                              b=to_device_matrix(np.require(b, requirements=["C", "W"]))
                              if not isinstance(b, torch.Tensor) else b, label=lab)

    if isinstance(source, GenerateSource):
        if source.n < 4:
            raise ValueError("need dimension >= 4")
        return (source.n, source.schedule.length,
                device_pencils(iter_generated_sequence(source.n, source.schedule, source.seed)))
    if isinstance(source, BaselineSource):
        dev = torch.cuda.current_device() if source.device else None
        return (source.n, source.length,
                device_pencils(iter_baseline_sequence(source.n, source.length, source.seed,
                                                      device=dev)))
    if isinstance(source, LoadSource):
        n, length, _ = pencil_io._manifest(source.directory)
        return n, length, device_pencils(pencil_io.iter_sequence(source.directory))
    raise TypeError(f"unknown sequence source {type(source).__name__}")


def run_experiment(spec):
    """The four-stage warm-start experiment over a whole sequence
    (harness.py:188-289), on the device.

    For every problem l = 2..N: (1) the dense solution of problem l-1 (the
    previous iteration's oracle: cuSOLVER zheevd of its standard form) gives
    the warm block — its lowest blk vectors, lambda_1 and lambda_{blk+1};
    (2) ChFSI from random vectors, rng (seed, l, 0); (3) ChFSI from the warm
    block, rng (seed, l, 1) — each ``repetitions`` times, the median wall time
    reported; (4) both converged results are checked against the dense
    spectrum of problem l (|dlambda| <= 1e-8 * scale, OracleMismatchError)
    and the tracked vectors of the two dense solutions are matched to give
    the median deviation angle. Pencils are streamed: only the previous
    problem's dense block lives across iterations.
    """
    if spec.solver in _OUT_OF_SCOPE:
        raise NotImplementedError(
            f"solver {spec.solver!r}: this package rebuilds the ChFSI path only; "
            "the LOBPCG baselines stay in the reference")
    from .analysis import match_eigenvectors

    with array_output("torch"):  # everything n-sized stays in HBM here
        n, length, pencils = _source_pencils(spec.source)
        cfg = ChfsiConfig(nev=spec.nev, **spec.solver_overrides)
        blk = cfg.resolve(n)[0]
        report = ExperimentReport(rows=[], n=n, length=length, solver=spec.solver, nev=spec.nev,
                                  blk=blk, repetitions=spec.repetitions,
                                  tracked_fraction=spec.tracked_fraction, seed=spec.seed)
        warnings = []
        if length < 2:
            warnings.append("sequence has a single problem; nothing to compare")
            report.warnings = warnings
            return report
        if blk >= n:
            raise ValueError(
                f"chfsi warm starts need blk < n for the window eigenvalue (blk={blk}, n={n})")
        tracked = max(1, int(np.ceil(spec.tracked_fraction * spec.nev)))
        keep = max(blk + 1, spec.nev)

        def cell(problem, guess, cell_seed, label):
            times, sol, rep = [], None, None
            for _ in range(spec.repetitions):
                sol, rep = chfsi_solve(problem.h, cfg, guess=guess,
                                       rng=np.random.default_rng(cell_seed), label=label)
                times.append(rep.wall_time)
            return sol, rep, statistics.median(times)

        it = iter(pencils)
        prev_sol, _, prev_vals = oracle_solve(next(it), keep)
        for pencil in it:
            sol_now, sp_now, vals_now = oracle_solve(pencil, keep)
            guess = ChfsiGuess(vectors=prev_sol.vectors[:, :blk], lambda1=float(prev_vals[0]),
                               lambda_blk_plus_1=float(prev_vals[blk]))
            lab = pencil.label
            del pencil
            sol_r, rep_r, t_r = cell(sp_now, None, (spec.seed, lab, 0), lab)
            sol_a, rep_a, t_a = cell(sp_now, guess, (spec.seed, lab, 1), lab)
            del sp_now, guess
            for rep, sol, start in ((rep_r, sol_r, "random"), (rep_a, sol_a, "approximate")):
                if rep.converged:
                    check_oracle(sol.values, vals_now, lab, start)
                else:
                    warnings.append(f"problem {lab}: {start} start did not converge")
            _, theta = match_eigenvectors(replace_tracked(prev_sol, tracked), None,
                                          replace_tracked(sol_now, tracked), None)
            report.rows.append(ExperimentRow(
                ell=lab, t_random_s=t_r, t_approx_s=t_a,
                speedup_time=t_r / t_a if t_a > 0 else float("inf"),
                matvecs_random=rep_r.matvecs, matvecs_approx=rep_a.matvecs,
                speedup_matvec=rep_r.matvecs / rep_a.matvecs if rep_a.matvecs else float("inf"),
                filtered_random=rep_r.filtered_vectors, filtered_approx=rep_a.filtered_vectors,
                inner_loops_random=rep_r.inner_loops, inner_loops_approx=rep_a.inner_loops,
                median_angle=float(np.median(theta)),
                max_residual_random=float(rep_r.final_residuals.max(initial=0.0)),
                max_residual_approx=float(rep_a.final_residuals.max(initial=0.0)),
                converged_random=rep_r.converged, converged_approx=rep_a.converged))
            prev_sol, prev_vals = sol_now, vals_now
        report.warnings = warnings
        return report


def _row_record(row):
    return {k: getattr(row, k) for k in REPORT_FIELDS}


def emit_report(report, fmt, path):
    """Write the rows as CSV (columns exactly REPORT_FIELDS) or as a JSON
    list of row objects (harness.py:316-336)."""
    path = Path(path)
    records = [_row_record(r) for r in report.rows]
    if fmt == "csv":
        with open(path, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=REPORT_FIELDS)
            w.writeheader()
            w.writerows(records)
    elif fmt == "json":
        with open(path, "w") as fh:
            json.dump(records, fh, indent=2)
    else:
        raise ValueError(f"unknown report format {fmt!r}")
