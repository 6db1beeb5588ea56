"""CPU baselines — TEST / MEASUREMENT INFRASTRUCTURE ONLY.

Only bench.py's cpu_baseline leg and its ``--impl reference`` arm (and tests)
may import this module; the product path never does.

The reference (pkg/src/tiledag) computes no numbers (pkg/README.md:11-12):
its CPU path is the schedule construction, ``tiledag.build_tree``
(qr.py:622-649), whose trace says which LAPACK tile kernel runs on which
tiles (qr.py:421-481) and, through its hazard DAG (taskgraph.py:262-322),
which may run concurrently — the runtime model of the thesis (PLASMA,
PAPER.md:2577-2585).  This module executes that trace on the host cores:

* ``DagReplay``: worker processes (one per core, OpenBLAS single-threaded
  inside each) run the LAPACK tile kernels of oracle/replay.py (dgeqrt,
  dgemqrt, dtpqrt, dtpmqrt) on tiles in shared (anonymous, fork-inherited) memory; the parent releases a
  task once its hazard-DAG predecessors are done (lowest trace id first).
  ``run_for(seconds)`` continues the same factorization, so successive
  bounded samples walk through the whole trace.
* ``time_dgeqrf``: numpy.linalg.qr(A, mode="r") — LAPACK dgeqrf, threaded
  OpenBLAS on every core — the best-effort CPU factorization.

scipy's LAPACK wrappers hold the GIL, hence processes, not threads.
"""
from __future__ import annotations

import heapq
import multiprocessing as mp
import os
import time
import mmap

import numpy as np

KIND_CODE = {"GEQRT": 0, "TTQRT": 1, "TSQRT": 2, "UNMQR": 3, "TTMQR": 4, "TSMQR": 5}  # include/tqr.h
WEIGHT = np.array([4, 2, 6, 6, 6, 12], dtype=np.float64)  # units of nb^3/3 flop (taskgraph.py:92-95)


def trace_arrays_of(build):
    """(kinds int8[n], idx int32[n,4] 1-based) of a QrBuild trace: the
    reference's (Task objects, qr.py:410-419) or this package's."""
    if hasattr(build, "trace_arrays"):
        k, i, _ = build.trace_arrays()
        return k, i
    tr = build.trace
    kinds = np.empty(len(tr), dtype=np.int8)
    idx = np.full((len(tr), 4), 0, dtype=np.int32)
    for t, task in enumerate(tr):
        kinds[t] = KIND_CODE[task.kind]
        ind = tuple(task.indices)
        idx[t, :len(ind)] = ind
    return kinds, idx


def edges_of(build, tiledag=None):
    """Hazard edges (u, v) of the build's trace: the reference's own
    build_from_trace when the reference module is given, else the build's."""
    if tiledag is not None:
        g = tiledag.build_from_trace(build.trace)
        return np.asarray([(u, v) for u, v, _ in g.edges], dtype=np.int64).reshape(-1, 2)
    return np.asarray([(u, v) for u, v, _ in build.hazard_edges()], dtype=np.int64).reshape(-1, 2)


# ---------------------------------------------------------------------------
# worker side


def _views(bufs, p, q, nb, ib):
    tiles = np.ndarray((p * q, nb, nb), dtype=np.float64, buffer=bufs[0])
    tg = np.ndarray((p * q, nb, ib), dtype=np.float64, buffer=bufs[1])
    te = np.ndarray((p * q, nb, ib), dtype=np.float64, buffer=bufs[2])
    # tile (i, j) 0-based at [j*p + i], stored transposed so that .T is the
    # Fortran-ordered nb x nb tile (T factors: Fortran ib x nb)
    return tiles, tg, te


def _worker(bufs, p, q, nb, ib, tasks, done):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from scipy.linalg import lapack as L

    tiles, tg, te = _views(bufs, p, q, nb, ib)
    T = lambda i, j: tiles[j * p + i].T  # noqa: E731  (Fortran-ordered view)
    TG = lambda i, k: tg[k * p + i].T  # noqa: E731
    TE = lambda i, k: te[k * p + i].T  # noqa: E731
    iu = np.triu_indices(nb)
    while True:
        msg = tasks.get()
        if msg is None:
            break
        tid, kd, a, b, c, d = msg
        if kd == 0:  # GEQRT(a, b)
            r, t, info = L.dgeqrt(ib, T(a, b))
            T(a, b)[...] = r
            TG(a, b)[...] = t
        elif kd == 3:  # UNMQR(a, b, c)
            r, info = L.dgemqrt(T(a, b), TG(a, b), T(a, c), side="L", trans="T")
            T(a, c)[...] = r
        elif kd in (1, 2):  # TTQRT / TSQRT (i=a, piv=b, k=c)
            l = nb if kd == 1 else 0
            rp, ri = T(b, c), T(a, c)
            x, y, t, info = L.dtpqrt(l, ib, np.triu(rp), np.triu(ri) if l else ri.copy(order="F"))
            rp[iu] = x[iu]
            if l:
                ri[iu] = y[iu]
            else:
                ri[...] = y
            TE(a, c)[...] = t
        else:  # TTMQR / TSMQR (i=a, piv=b, k=c, j=d)
            l = nb if kd == 4 else 0
            v = np.triu(T(a, c)) if l else T(a, c)
            x, y, info = L.dtpmqrt(l, v, TE(a, c), T(b, d), T(a, d), side="L", trans="T")
            T(b, d)[...] = x
            T(a, d)[...] = y
        done.put(tid)


# ---------------------------------------------------------------------------
# parent side


class DagReplay:
    """Parallel LAPACK replay of a tiled-QR trace over its hazard DAG."""

    def __init__(self, A, p, q, nb, kinds, idx, edges, workers=None, ib=32):
        self.p, self.q, self.nb, self.ib = p, q, nb, ib
        self.kinds = np.asarray(kinds, dtype=np.int64)
        self.idx = np.asarray(idx, dtype=np.int64) - 1
        n = len(self.kinds)
        self.n = n
        self.flops = WEIGHT[self.kinds] * nb ** 3 / 3.0
        self.workers = workers or os.cpu_count() or 1
        sizes = [p * q * nb * nb * 8, p * q * ib * nb * 8, p * q * ib * nb * 8]
        # anonymous MAP_SHARED memory, inherited by the forked workers (no
        # /dev/shm size limit involved)
        self.bufs = [mmap.mmap(-1, max(s, 8)) for s in sizes]
        self.tiles = np.ndarray((p * q, nb, nb), dtype=np.float64, buffer=self.bufs[0])
        # successor CSR and in-degrees
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        order = np.argsort(e[:, 0], kind="stable")
        self.succ = e[order, 1]
        self.succ_ptr = np.searchsorted(e[order, 0], np.arange(n + 1))
        self.indeg0 = np.bincount(e[:, 1], minlength=n).astype(np.int64)
        ctx = mp.get_context("fork")
        self.tq, self.dq = ctx.Queue(), ctx.Queue()
        self.procs = [ctx.Process(target=_worker, args=(self.bufs, p, q, nb, ib, self.tq, self.dq), daemon=True)
                      for _ in range(self.workers)]
        for pr in self.procs:
            pr.start()
        self.reload(A)

    def reload(self, A):
        """Start a fresh factorization of A (the previous one completed)."""
        p, q, nb = self.p, self.q, self.nb
        for j in range(q):
            for i in range(p):
                self.tiles[j * p + i] = A[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb].T
        self.reset()

    def reset(self):
        self.indeg = self.indeg0.copy()
        self.ready = [t for t in range(self.n) if self.indeg[t] == 0]
        heapq.heapify(self.ready)
        self.inflight = 0
        self.completed = 0

    def _issue(self):
        while self.ready and self.inflight < 2 * self.workers:
            t = heapq.heappop(self.ready)
            a, b, c, d = (int(x) for x in self.idx[t])
            self.tq.put((t, int(self.kinds[t]), a, b, c, d))
            self.inflight += 1

    def run_for(self, seconds):
        """Continue the factorization for ~seconds; returns (flops, elapsed,
        tasks completed in this window).  In-flight tasks are drained before
        returning, so the window's flops are exactly its completed tasks."""
        t0 = time.perf_counter()
        fl, cnt = 0.0, 0
        stop = False
        self._issue()
        while self.inflight:
            t = self.dq.get()
            self.inflight -= 1
            fl += self.flops[t]
            cnt += 1
            self.completed += 1
            for s in self.succ[self.succ_ptr[t]:self.succ_ptr[t + 1]]:
                self.indeg[s] -= 1
                if self.indeg[s] == 0:
                    heapq.heappush(self.ready, int(s))
            if not stop and time.perf_counter() - t0 >= seconds:
                stop = True
            if not stop:
                self._issue()
        return fl, time.perf_counter() - t0, cnt

    def finished(self):
        return self.completed >= self.n

    def close(self):
        for _ in self.procs:
            self.tq.put(None)
        for pr in self.procs:
            pr.join(timeout=10)
        self.tiles = None


def time_dgeqrf(A, threads=None):
    """numpy.linalg.qr(A, mode='r') (LAPACK dgeqrf) on every core:
    (seconds, GFLOP/s at 2n^2(m-n/3), threads)."""
    from threadpoolctl import threadpool_limits
    m, n = A.shape
    th = threads or os.cpu_count() or 1
    with threadpool_limits(th):
        t0 = time.perf_counter()
        np.linalg.qr(A, mode="r")
        dt = time.perf_counter() - t0
    return dt, 2.0 * n * n * (m - n / 3.0) / dt / 1e9, th


def load_reference():
    """The reference package (baseline/_ref install, or the read-only source
    tree in the build container); None if absent."""
    import importlib
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for path in (os.path.join(root, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "tiledag")):
            if path not in sys.path:
                sys.path.insert(0, path)
            return importlib.import_module("tiledag")
    return None
