"""Kernel tags, tile/task records and weight models of the tiled QR path.

Mirrors the pieces of the reference's core engine that the QR path uses
(pkg/src/tiledag/taskgraph.py): the kernel tags (:19-40), TileRef (:48-54),
Task (:57-75), WeightModel (:78-146) and the hazard DAG of a QR trace
(build_from_trace, :262-322) with Backflow/earliest times (annotate_cp,
:338-362).  Hazard edges always come from the C++ schedule compiler (the
same edges drive the device dependency counters), for this package's traces
and for the reference's own Task lists alike.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

GEQRT = "GEQRT"
TSQRT = "TSQRT"
TTQRT = "TTQRT"
UNMQR = "UNMQR"
TSMQR = "TSMQR"
TTMQR = "TTMQR"
POTRF, TRSM, SYRK, GEMM, TRTRI, TRMM, LAUUM = "POTRF", "TRSM", "SYRK", "GEMM", "TRTRI", "TRMM", "LAUUM"
GEADD, COPY, BARRIER = "GEADD", "COPY", "BARRIER"

ALL_KINDS = frozenset({POTRF, TRSM, SYRK, GEMM, TRTRI, TRMM, LAUUM, GEQRT, TSQRT, TTQRT,
                       UNMQR, TSMQR, TTMQR, GEADD, COPY, BARRIER})
# order of the C ABI's enum tqr_kind (include/tqr.h)
QR_KINDS = (GEQRT, TTQRT, TSQRT, UNMQR, TTMQR, TSMQR)

RAW, WAR, WAW, EXPLICIT = "RAW", "WAR", "WAW", "EXPLICIT"
_CAUSE = (RAW, WAR, WAW)


class TileRef(NamedTuple):
    matrix: str
    row: int
    col: int


class Task:
    """One kernel invocation on tiles; `id` is its position in the trace."""

    __slots__ = ("id", "kind", "indices", "reads", "writes")

    def __init__(self, id, kind, indices=(), reads=(), writes=()):
        self.id = id
        self.kind = kind
        self.indices = tuple(indices)
        self.reads = tuple(reads)
        self.writes = tuple(writes)

    def __repr__(self):
        return f"{self.kind}({','.join(str(i) for i in self.indices)})#{self.id}"


def qr_task(tid, kind, idx):
    """Task with the symbolic read/write sets of qr.py:421-481."""
    if kind == GEQRT:
        i, k = idx
        return Task(tid, kind, idx, (TileRef("D", i, k),), (TileRef("R", i, k), TileRef("V", i, k)))
    if kind == UNMQR:
        i, k, j = idx
        return Task(tid, kind, idx, (TileRef("V", i, k), TileRef("D", i, j)), (TileRef("D", i, j),))
    if kind == TTQRT:
        i, piv, k = idx
        return Task(tid, kind, idx, (TileRef("R", i, k), TileRef("R", piv, k)),
                    (TileRef("R", piv, k), TileRef("T", i, k)))
    if kind == TSQRT:
        i, piv, k = idx
        return Task(tid, kind, idx, (TileRef("D", i, k), TileRef("R", piv, k)),
                    (TileRef("R", piv, k), TileRef("S", i, k)))
    i, piv, k, j = idx
    m = "T" if kind == TTMQR else "S"
    return Task(tid, kind, idx, (TileRef(m, i, k), TileRef("D", i, j), TileRef("D", piv, j)),
                (TileRef("D", i, j), TileRef("D", piv, j)))


class WeightModel:
    """Integer kernel durations; one unit is nb^3/3 flops (taskgraph.py:78-146)."""

    CHOLESKY = {POTRF: 1, TRSM: 3, SYRK: 3, GEMM: 6, TRTRI: 1, TRMM: 3, LAUUM: 1, COPY: 0, BARRIER: 0}
    QR = {GEQRT: 4, TTQRT: 2, UNMQR: 6, TTMQR: 6, TSQRT: 6, TSMQR: 12, BARRIER: 0}

    def __init__(self, mode="unit", table=None):
        if mode == "unit":
            table = {k: 1 for k in ALL_KINDS}
            table[BARRIER] = 0
            table[COPY] = 0
        elif mode == "cholesky":
            table = dict(self.CHOLESKY)
        elif mode in ("qr-tt", "qr-full"):
            table = dict(self.QR)
        elif mode == "custom":
            table = dict(table or {})
        else:
            raise ValueError(f"unknown weight mode {mode!r}")
        for kind, w in table.items():
            if kind not in ALL_KINDS:
                raise ValueError(f"unknown kernel kind {kind!r}")
            if not isinstance(w, int) or w < 0:
                raise ValueError(f"weight of {kind} must be a nonnegative integer")
        table[BARRIER] = 0
        self.mode = mode
        self.table = table

    @classmethod
    def unit(cls):
        return cls("unit")

    @classmethod
    def cholesky(cls):
        return cls("cholesky")

    @classmethod
    def qr_tt(cls):
        return cls("qr-tt")

    @classmethod
    def qr_full(cls):
        return cls("qr-full")

    @classmethod
    def custom(cls, table):
        return cls("custom", table)

    def __getitem__(self, kind):
        try:
            return self.table[kind]
        except KeyError:
            raise KeyError(f"weight model {self.mode!r} has no weight for {kind}") from None

    def of(self, task):
        return self[task.kind]

    def qr_vector(self):
        """Weights by C-ABI kind order, -1 where the model lacks the kind."""
        return [int(self.table.get(k, -1)) for k in QR_KINDS]


@dataclass
class CpAnnotation:
    priority: dict
    cp_length: int
    earliest: dict
    latest: dict

    def critical_ids(self):
        return [i for i in self.priority if self.earliest[i] == self.latest[i]]


class TaskGraph:
    """Hazard DAG over a trace; edges (u, v, cause) with u < v."""

    def __init__(self, tasks, edges):
        self.tasks = list(tasks)
        self.edges = list(edges)
        self._succ = None
        self._pred = None

    def __len__(self):
        return len(self.tasks)

    def successors(self):
        if self._succ is None:
            succ = {t.id: [] for t in self.tasks}
            for u, v, _ in self.edges:
                succ[u].append(v)
            self._succ = succ
        return self._succ

    def predecessors(self):
        if self._pred is None:
            pred = {t.id: [] for t in self.tasks}
            for u, v, _ in self.edges:
                pred[v].append(u)
            self._pred = pred
        return self._pred

    def topo_order(self):
        return [t.id for t in self.tasks]  # trace-built: edges go forward


def _trace_edges(trace):
    """Hazard edges of any QR trace (this package's or the reference's Task
    objects: .id .kind .indices), computed by the C++ compiler
    (tqr_trace_build + tqr_build_hazard_edges, the rule of
    taskgraph.py:262-322)."""
    import ctypes as C

    import numpy as np

    from . import _lib

    tasks = list(trace)
    n = len(tasks)
    kind = np.empty(max(n, 1), dtype=np.int8)
    idx = np.full((max(n, 1), 4), -1, dtype=np.int32)
    code = {k: c for c, k in enumerate(QR_KINDS)}
    p = q = 1
    for t, task in enumerate(tasks):
        if task.kind not in code:
            raise ValueError(f"build_from_trace: {task.kind} is not a QR kernel")
        kind[t] = code[task.kind]
        ind = tuple(task.indices)
        idx[t, :len(ind)] = ind
        rows = ind[:1] if task.kind in (GEQRT, UNMQR) else ind[:2]
        p = max(p, *rows)
        q = max(q, ind[-1])
    h = C.c_void_p()
    L = _lib.lib()
    _lib.check(L.tqr_trace_build(p, q, kind.ctypes.data_as(_lib.i8p), _lib.ptr_i32(idx), n, C.byref(h)))
    try:
        cnt = C.c_int64()
        _lib.check(L.tqr_build_hazard_edges(h, None, 0, C.byref(cnt)))
        e = np.empty((max(cnt.value, 1), 3), dtype=np.int32)
        _lib.check(L.tqr_build_hazard_edges(h, _lib.ptr_i32(e), cnt.value, C.byref(cnt)))
    finally:
        L.tqr_build_free(h)
    ids = [t.id for t in tasks]
    cause = (RAW, WAR, WAW)
    return [(ids[u], ids[v], cause[c]) for u, v, c in e[:cnt.value].tolist()]


def build_from_trace(trace) -> TaskGraph:
    """Hazard DAG of a QR trace (taskgraph.py:262-322): a QrBuild's trace uses
    its compiled edges (the ones the device runs on), any other QR trace —
    e.g. the reference's own Task list — goes through the same C++ rule."""
    build = getattr(trace, "build", None)
    if build is not None:
        return TaskGraph(trace, build.hazard_edges())
    return TaskGraph(trace, _trace_edges(trace))


def annotate_cp(graph: TaskGraph, weights: WeightModel) -> CpAnnotation:
    """Backflow priorities and earliest starts (taskgraph.py:338-362)."""
    w = {t.id: weights.of(t) for t in graph.tasks}
    succ, pred = graph.successors(), graph.predecessors()
    order = graph.topo_order()
    priority = {}
    for u in reversed(order):
        best = 0
        for v in succ[u]:
            if priority[v] > best:
                best = priority[v]
        priority[u] = w[u] + best
    cp_length = max(priority.values(), default=0)
    earliest = {}
    for u in order:
        est = 0
        for v in pred[u]:
            f = earliest[v] + w[v]
            if f > est:
                est = f
        earliest[u] = est
    latest = {u: cp_length - priority[u] for u in priority}
    return CpAnnotation(priority, cp_length, earliest, latest)


def asap_times(trace, weights: WeightModel):
    """(finish by id, cp) on unbounded processors, via the hazard DAG."""
    g = build_from_trace(trace)
    ann = annotate_cp(g, weights)
    fins = {t.id: ann.earliest[t.id] + weights.of(t) for t in g.tasks}
    return fins, max(fins.values(), default=0)


def trace_cp(trace, weights: WeightModel) -> int:
    return asap_times(trace, weights)[1]


def t_seq(trace, weights: WeightModel) -> int:
    return sum(weights.of(t) for t in trace)
