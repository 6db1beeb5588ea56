"""Elimination lists, coarse tables and the tiled TT/TS builder — the
reference's QR entry points (pkg/src/tiledag/qr.py), backed by the C++
schedule compiler in libtqr.so (csrc/sched.cpp).

Every function keeps the reference signature, return types, error classes
and messages, so code written against ``tiledag`` runs unchanged; results
are bit-exact with the reference (tests/test_schedule_parity.py).  The
numeric engine (``tiled_qr``, engine.py) consumes the same QrBuild objects.
Rows and columns are 1-based (qr.py:11).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from math import ceil

import numpy as np

from . import _lib
from ._lib import check, lib, ptr_i32, ptr_i64
from .taskgraph import (GEQRT, QR_KINDS, TSMQR, TSQRT, TTMQR, TTQRT, UNMQR,
                        WeightModel, qr_task)

COARSE_ALGOS = ("sameh-kuck", "fibonacci", "greedy")
TREE_ALGOS = ("flattree", "fibonacci", "greedy", "binarytree", "plasmatree", "asap", "grasap")


@dataclass(frozen=True)
class ElimEntry:
    """elim(i, piv, k): zero tile (i,k) by combining rows i and piv (qr.py:31-38)."""

    i: int
    piv: int
    k: int
    step: int = 0


def _to_array(entries):
    """(n, 4) int32 (i, piv, k, step) of any iterable of entries exposing
    .i .piv .k (and optionally .step) — this package's ElimEntry or the
    reference's (qr.py:31-38)."""
    rows = [(e.i, e.piv, e.k, getattr(e, "step", 0)) for e in entries]
    a = np.empty((len(rows), 4), dtype=np.int32)
    if rows:
        a[:] = rows
    return a


def elim_array(elim):
    """(n, 4) int32 array of any elimination list: this package's
    EliminationList or one duck-typed like the reference's (``.p .q`` plus
    iteration over entries, qr.py:41-55)."""
    return _to_array(list(elim))


def _validate_any(elim):
    """EliminationList.validate() semantics (qr.py:56-83) for any list-like
    object, run by the C++ validator (same messages)."""
    a = elim_array(elim)
    msg = C.create_string_buffer(512)
    rc = lib().tqr_elim_validate(int(elim.p), int(elim.q), ptr_i32(a), len(a), msg, 512)
    if rc == 1:
        raise ValueError(msg.value.decode())
    check(rc)
    return True


def _from_array(a):
    return [ElimEntry(int(i), int(v), int(k), int(s)) for i, v, k, s in a.tolist()]


class EliminationList:
    """Ordered eliminations zeroing every sub-diagonal tile (qr.py:41-141)."""

    def __init__(self, p, q, entries):
        self.p = p
        self.q = q
        self.entries = list(entries)

    def __iter__(self):
        return iter(self.entries)

    def __len__(self):
        return len(self.entries)

    def array(self):
        """(n, 4) int32 array of (i, piv, k, step)."""
        return _to_array(self.entries)

    def validate(self):
        return _validate_any(self)

    def normalized(self):
        a = self.array()
        out = np.empty_like(a)
        check(lib().tqr_elim_normalized(self.p, self.q, ptr_i32(a), len(a), ptr_i32(out)))
        return EliminationList(self.p, self.q, _from_array(out))

    def with_steps(self):
        a = self.array()
        out = np.empty_like(a)
        check(lib().tqr_elim_with_steps(ptr_i32(a), len(a), ptr_i32(out)))
        return EliminationList(self.p, self.q, _from_array(out))

    def to_csv(self):
        lines = ["k,i,piv,step"]
        lines += [f"{e.k},{e.i},{e.piv},{e.step}" for e in self.entries]
        return "\n".join(lines) + "\n"

    @classmethod
    def from_csv(cls, p, q, text):
        entries = []
        for line in text.strip().splitlines()[1:]:
            k, i, piv, step = (int(x) for x in line.split(","))
            entries.append(ElimEntry(i, piv, k, step))
        return cls(p, q, entries)


class CoarseTable:
    """coarse(i,k): unit-cost step at which tile (i,k) is zeroed (qr.py:144-197)."""

    def __init__(self, p, q, steps, algo="", x=None):
        self.p = p
        self.q = q
        self.steps = dict(steps)
        self.algo = algo
        self.x = x

    def __call__(self, i, k):
        return self.steps[(i, k)]

    def cp(self):
        return max(self.steps.values(), default=0)

    def groups(self):
        g = {}
        for (i, k), s in self.steps.items():
            g.setdefault((s, k), []).append(i)
        return {key: sorted(rows) for key, rows in g.items()}

    def validate(self, elim: EliminationList):
        for e in elim:
            s = self.steps[(e.i, e.k)]
            if e.k > 1:
                if self.steps[(e.i, e.k - 1)] >= s:
                    raise ValueError(f"coarse dependency violated: own row at ({e.i},{e.k})")
                if e.piv > e.k - 1 and self.steps[(e.piv, e.k - 1)] >= s:
                    raise ValueError(f"coarse dependency violated: pivot row at ({e.i},{e.k})")
        for k in range(1, min(self.p, self.q) + 1):
            col = [self.steps[(i, k)] for i in range(k + 1, self.p + 1)]
            if self.algo == "sameh-kuck":
                ok = all(a < b for a, b in zip(col, col[1:]))
            else:
                ok = all(a >= b for a, b in zip(col, col[1:]))
            if not ok:
                raise ValueError(f"column {k} violates the {self.algo} sweep order")
        return True

    def to_csv(self):
        lines = ["i\\k," + ",".join(str(k) for k in range(1, self.q + 1))]
        for i in range(1, self.p + 1):
            lines.append(f"{i}," + ",".join(str(self.steps.get((i, k), "")) for k in range(1, self.q + 1)))
        return "\n".join(lines) + "\n"


def fibonacci_x(p):
    """Least x with x(x+1)/2 >= p-1 (qr.py:200-205)."""
    x = 0
    while x * (x + 1) // 2 < p - 1:
        x += 1
    return x


def coarse_schedule(p, q, algo):
    """Coarse table + elimination list of Sameh-Kuck, Fibonacci or Greedy
    (qr.py:279-297)."""
    if not (p >= q >= 1):
        raise ValueError("need p >= q >= 1")
    algo_l = algo.lower()
    n = sum(p - k for k in range(1, min(p, q) + 1))
    steps = np.zeros(p * q, dtype=np.int32)
    elim = np.empty((max(n, 1), 4), dtype=np.int32)
    n_out, x_out = C.c_int64(), C.c_int32()
    check(lib().tqr_coarse_schedule(p, q, algo_l.encode(), ptr_i32(steps), ptr_i32(elim), n,
                                    C.byref(n_out), C.byref(x_out)))
    st = steps.reshape(p, q)
    ii, kk = np.nonzero(st)
    table_steps = {(int(i) + 1, int(k) + 1): int(st[i, k]) for i, k in zip(ii.tolist(), kk.tolist())}
    name = "sameh-kuck" if algo_l in ("sameh-kuck", "samehkuck", "flattree") else algo_l
    table = CoarseTable(p, q, table_steps, name, int(x_out.value))
    return table, EliminationList(p, q, _from_array(elim[:n_out.value]))


def eager_coarse(elim: EliminationList) -> CoarseTable:
    """Dependence-driven re-execution of a list (qr.py:300-307)."""
    steps = {(e.i, e.k): e.step for e in elim.with_steps()}
    return CoarseTable(elim.p, elim.q, steps, "eager")


def coarse_cp_oracle(p, q, algo):
    """Closed-form coarse critical paths (qr.py:310-327)."""
    if not (p >= q >= 1):
        raise ValueError("need p >= q >= 1")
    algo = algo.lower()
    if algo in ("sameh-kuck", "samehkuck", "flattree"):
        if p == q:
            return 2 * q - 3 if q > 1 else 0
        return p + q - 2
    if algo == "fibonacci":
        x = fibonacci_x(p)
        if p == q:
            return x + 2 * q - 4 if q > 1 else 0
        return x + 2 * q - 2
    if algo == "greedy":
        return coarse_schedule(p, q, "greedy")[0].cp()
    raise ValueError(f"unknown coarse algorithm {algo!r}")


def flat_tree_list(p, q):
    return coarse_schedule(p, q, "sameh-kuck")[1]


def plasmatree_list(p, q, bs):
    """PLASMA domains of bs rows + binary merge of heads (qr.py:336-362)."""
    n = C.c_int64()
    cap = sum(p - k for k in range(1, min(p, q) + 1)) if p >= 1 else 0
    out = np.empty((max(cap, 1), 4), dtype=np.int32)
    check(lib().tqr_plasmatree_list(p, q, int(bs), ptr_i32(out), cap, C.byref(n)))
    return EliminationList(p, q, _from_array(out[:n.value]))


def binary_tree_list(p, q):
    return plasmatree_list(p, q, 1)


# ---------------------------------------------------------------------------
# tiled builder


class _Trace(list):
    """The Task trace of a QrBuild (a list), remembering its build so the
    hazard DAG comes from the C++ compiler."""

    build = None


class QrBuild:
    """Tiled QR task graph with weighted ASAP times (qr.py:376-532).

    Attributes mirror the reference: p q family weights trace zeroed updates
    cp counts total_weight elim.  The C++ build is kept in ``_h`` so the
    numeric engine can compile it into a device schedule.
    """

    def __init__(self, p, q, family="TT", weights=None, keep_trace=True, record_updates=False):
        if not (p >= q >= 1):
            raise ValueError("need p >= q >= 1")
        if family not in ("TT", "TS"):
            raise ValueError("kernel family must be 'TT' or 'TS'")
        self.p, self.q, self.family = p, q, family
        self.weights = weights if weights is not None else WeightModel.qr_tt()
        self.keep_trace = keep_trace
        self.record_updates = record_updates
        self.trace = [] if keep_trace else None
        self.zeroed, self.updates = {}, {}
        self.cp = 0
        self.counts = {GEQRT: 0, TTQRT: 0, TSQRT: 0, UNMQR: 0, TTMQR: 0, TSMQR: 0}
        self.total_weight = 0
        self.elim = None
        self._h = None
        self._trace = None

    # -- C++ handle ---------------------------------------------------------

    def _adopt(self, handle, elim=None):
        if self._h is not None:
            lib().tqr_build_free(self._h)
        self._h = handle
        info = _lib.BuildInfo()
        check(lib().tqr_build_get_info(handle, C.byref(info)))
        self.cp = int(info.cp)
        self.total_weight = int(info.total_weight)
        self.counts = {GEQRT: 0, TTQRT: 0, TSQRT: 0, UNMQR: 0, TTMQR: 0, TSMQR: 0}
        for t, k in enumerate(QR_KINDS):
            self.counts[k] = int(info.counts[t])
        z = np.empty((max(info.n_zeroed, 1), 3), dtype=np.int64)
        check(lib().tqr_build_get_zeroed(handle, ptr_i64(z)))
        self.zeroed = {(i, k): v for i, k, v in z[:info.n_zeroed].tolist()}
        self.updates = {}
        if self.record_updates and info.n_updates:
            u = np.empty((info.n_updates, 4), dtype=np.int64)
            check(lib().tqr_build_get_updates(handle, ptr_i64(u)))
            for i, k, j, fin in u.tolist():
                self.updates.setdefault((i, k), {})[j] = fin
        if elim is None:
            e = np.empty((max(info.n_elim, 1), 4), dtype=np.int32)
            check(lib().tqr_build_get_elim(handle, ptr_i32(e)))
            elim = EliminationList(self.p, self.q, _from_array(e[:info.n_elim]))
        self.elim = elim
        self._n_trace = int(info.n_trace)
        self._trace = None
        if self.keep_trace:
            self.__dict__.pop("trace", None)
        return self

    def __getattr__(self, name):
        if name == "trace":  # materialized lazily: O(tasks) Python objects
            if not self.__dict__.get("keep_trace", False):
                return None
            tr = _Trace(qr_task(t, kind, idx) for t, (kind, idx) in enumerate(self.trace_arrays_iter()))
            tr.build = self
            self.__dict__["trace"] = tr
            return tr
        raise AttributeError(name)

    def __del__(self):
        h = self.__dict__.get("_h")
        try:
            if h is not None and _lib._lib is not None:
                _lib._lib.tqr_build_free(h)
        except (AttributeError, TypeError):  # interpreter shutdown: modules already torn down
            pass

    def trace_arrays(self):
        """(kind int8[n], idx int32[n,4], finish int64[n]) of the trace."""
        if self._h is None:
            raise RuntimeError("QrBuild has no compiled trace (run_list first)")
        n = self._n_trace
        kind = np.empty(max(n, 1), dtype=np.int8)
        idx = np.empty((max(n, 1), 4), dtype=np.int32)
        fin = np.empty(max(n, 1), dtype=np.int64)
        check(lib().tqr_build_get_trace(self._h, kind.ctypes.data_as(_lib.i8p), ptr_i32(idx), ptr_i64(fin)))
        return kind[:n], idx[:n], fin[:n]

    def trace_arrays_iter(self):
        kind, idx, _ = self.trace_arrays()
        arity = (2, 3, 3, 3, 4, 4)
        for kd, row in zip(kind.tolist(), idx.tolist()):
            yield QR_KINDS[kd], tuple(row[:arity[kd]])

    def hazard_edges(self):
        """build_from_trace edges of the trace (taskgraph.py:262-322)."""
        n = C.c_int64()
        check(lib().tqr_build_hazard_edges(self._h, None, 0, C.byref(n)))
        e = np.empty((max(n.value, 1), 3), dtype=np.int32)
        check(lib().tqr_build_hazard_edges(self._h, ptr_i32(e), n.value, C.byref(n)))
        cause = ("RAW", "WAR", "WAW")
        return [(u, v, cause[c]) for u, v, c in e[:n.value].tolist()]

    def run_list(self, elim: EliminationList):
        """Tiled translation of ``elim`` (qr.py:520-532): this package's
        EliminationList or the reference's (entries read as .i .piv .k)."""
        a = elim_array(elim)
        h = C.c_void_p()
        w = _weights_arg(self.weights)
        check(lib().tqr_tiled_build(self.p, self.q, ptr_i32(a), len(a), int(self.family == "TS"), ptr_i64(w),
                                    int(self.keep_trace), int(self.record_updates), 0, C.byref(h)))
        return self._adopt(h, elim)


def _weights_arg(weights):
    """Per-kind weight vector (C-ABI kind order, -1 where the model has no
    weight) of this package's WeightModel or any model answering
    ``weights[kind]`` / raising KeyError like the reference's
    (taskgraph.py:139-146)."""
    if weights is None:
        weights = WeightModel.qr_tt()
    if hasattr(weights, "qr_vector"):
        return np.asarray(weights.qr_vector(), dtype=np.int64)
    w = []
    for k in QR_KINDS:
        try:
            w.append(int(weights[k]))
        except KeyError:
            w.append(-1)
    return np.asarray(w, dtype=np.int64)


def tiled_build(elim: EliminationList, family="TT", weights=None, keep_trace=True,
                record_updates=False, validate=True) -> QrBuild:
    """Tiled translation of any valid elimination list (qr.py:535-540); the
    list may be the reference's own EliminationList (duck-typed)."""
    if validate:
        _validate_any(elim)
    b = QrBuild(elim.p, elim.q, family, weights, keep_trace, record_updates)
    return b.run_list(elim)


def tiled_graph(elim: EliminationList, family="TT"):
    return tiled_build(elim, family).trace


def _tree(p, q, algo, family, bs, grasap_i, weights, keep_trace, record_updates):
    h = C.c_void_p()
    w = _weights_arg(weights)
    check(lib().tqr_build_tree(p, q, algo.encode(), int(family != "TT"),
                               _lib.TQR_NO_BS if bs is None else int(bs), int(grasap_i), ptr_i64(w),
                               int(keep_trace), int(record_updates), C.byref(h)))
    if family not in ("TT", "TS"):
        lib().tqr_build_free(h)
        raise ValueError("kernel family must be 'TT' or 'TS'")
    b = QrBuild(p, q, family, weights, keep_trace, record_updates)
    return b._adopt(h)


def asap_build(p, q, weights=None, keep_trace=True, record_updates=False) -> QrBuild:
    """Event-driven Asap over TT kernels (qr.py:586-592)."""
    return _tree(p, q, "asap", "TT", None, 1, weights, keep_trace, record_updates)


def grasap_build(p, q, i=1, weights=None, keep_trace=True, record_updates=False) -> QrBuild:
    """Greedy on the first q-i columns, Asap on the trailing i (qr.py:595-611)."""
    if not (1 <= i <= q):
        raise ValueError("need 1 <= i <= q")
    return _tree(p, q, "grasap", "TT", None, i, weights, keep_trace, record_updates)


def asap_graph(p, q):
    return asap_build(p, q).trace


def grasap_graph(p, q, i=1):
    return grasap_build(p, q, i).trace


def build_tree(p, q, algo, family="TT", bs=None, grasap_i=1, weights=None,
               keep_trace=True, record_updates=False) -> QrBuild:
    """One-stop construction of any studied elimination tree (qr.py:622-649)."""
    return _tree(p, q, algo, family, bs, grasap_i, weights, keep_trace, record_updates)


def zeroed_table_csv(build: QrBuild):
    lines = ["i\\k," + ",".join(str(k) for k in range(1, build.q + 1))]
    for i in range(1, build.p + 1):
        lines.append(f"{i}," + ",".join(str(build.zeroed.get((i, k), "")) for k in range(1, build.q + 1)))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# closed forms and conservation (qr.py:663-742)


def total_weight(p, q):
    if not (p >= q >= 1):
        raise ValueError("need p >= q >= 1")
    return 6 * p * q * q - 2 * q ** 3


def verify_weight(build: QrBuild):
    return build.total_weight == total_weight(build.p, build.q)


def elim_weight(q, k):
    return 10 + 18 * (q - k)


def qr_flops(m, n):
    """Algorithmic flops of the factorization, 2 n^2 (m - n/3): the metric's
    numerator; equals total_weight(p, q) * nb^3 / 3 for m = p nb, n = q nb."""
    return 2.0 * n * n * (m - n / 3.0)


def flattree_cp_oracle(p, q):
    if not (p >= q >= 1):
        raise ValueError("need p >= q >= 1")
    if q == 1:
        return 2 * p + 2
    if p == q:
        return 22 * p - 24
    return 6 * p + 16 * q - 22


def sk_coarse_closed_form(p, q):
    if q < 1 or (p == q == 1):
        return 0
    if p == q:
        return 2 * p - 3
    return p + q - 2


def flattree_cp_composed(p, q):
    c1 = sk_coarse_closed_form(p, q - 1)
    c2 = sk_coarse_closed_form(p, q)
    return 10 * (q - 1) + 6 * c1 + 4 + 2 * (c2 - c1)


def fibonacci_cp_bounds(p, q):
    if not (p >= q >= 1):
        raise ValueError("need p >= q >= 1")
    return 22 * q - 30, 22 * q + 6 * ceil((2 * p) ** 0.5)


def tiled_translation(i, k, coarse: CoarseTable):
    if k >= coarse.q:
        raise ValueError("translation excludes the last column (need k <= q-1)")
    if not (i > k >= 1):
        raise ValueError("need a sub-diagonal tile")
    return 10 * k + 6 * coarse(i, k)
