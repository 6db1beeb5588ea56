"""Numeric tiled QR on B200 (no reference counterpart: the reference runs no
kernels, pkg/README.md:11-12).

``tiled_qr(A, nb, algo=...)`` factors an m x n fp64 matrix with the tiled
TT/TS kernels in the order fixed by the reference elimination tree
(build_tree, qr.py:622-649; or any user list via tiled_build,
qr.py:535-540).  Device memory and streams come from PyTorch; every kernel
is in libtqr.so (csrc/).  There is no CPU fallback: without CUDA or without
the library this module raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import torch

from . import _lib
from ._lib import check, lib
from .qr import QrBuild, build_tree, tiled_build


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _vp(t):
    return C.c_void_p(t.data_ptr())


class Plan:
    """A QrBuild compiled into a static device schedule for tile size nb
    (tqr_plan_create).  Reusable across matrices of the same shape."""

    IO_IN, IO_OUT = 1, 2

    def __init__(self, build: QrBuild, nb=256, ib=32, io=0):
        """io: 0 for device-resident input/output, or IO_IN | IO_OUT to
        compile PACK / UNPACK work items that overlap the host transfers
        with the factorization (factor_stream)."""
        if not torch.cuda.is_available():
            raise RuntimeError("tiled QR needs a CUDA device (no CPU fallback)")
        if build._h is None or not build.keep_trace:
            raise ValueError("the plan needs a QrBuild made with keep_trace=True")
        self.build = build
        self.io = int(io)
        h = C.c_void_p()
        check(lib().tqr_plan_create_io(build._h, int(nb), int(ib), self.io, C.byref(h)))
        self._h = h
        info = _lib.PlanInfo()
        check(lib().tqr_plan_get_info(h, C.byref(info)))
        self.info = info
        self.p, self.q, self.nb, self.ib = info.p, info.q, info.nb, info.ib
        self.m, self.n = self.p * self.nb, self.q * self.nb
        self.flops = float(info.flops_alg)

    def __del__(self):
        h = self.__dict__.get("_h")
        try:
            if h is not None and _lib._lib is not None:
                _lib._lib.tqr_plan_free(h)
        except (AttributeError, TypeError):  # interpreter shutdown: modules already torn down
            pass

    def alloc(self, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        tiles = torch.empty(self.p * self.q * self.nb * self.nb, dtype=torch.float64, device=dev)
        tg = torch.zeros(self.p * self.q * self.info.tg_stride, dtype=torch.float64, device=dev)
        te = torch.zeros(self.p * self.q * self.info.te_stride, dtype=torch.float64, device=dev)
        return tiles, tg, te

    def pack(self, A, tiles, stream=None):
        """Row-major (C-contiguous) or column-major m x n device matrix -> tiles."""
        assert A.dtype == torch.float64 and A.is_cuda and A.shape == (self.m, self.n)
        if A.is_contiguous():
            check(lib().tqr_pack(_vp(A), A.stride(0), 1, _vp(tiles), self.p, self.q, self.nb, _stream_ptr(stream)))
        elif A.t().is_contiguous():
            check(lib().tqr_pack(_vp(A), A.stride(1), 0, _vp(tiles), self.p, self.q, self.nb, _stream_ptr(stream)))
        else:
            raise ValueError("A must be row- or column-major contiguous")

    def factor(self, tiles, tg, te, stream=None):
        check(lib().tqr_factor(self._h, _vp(tiles), _vp(tg), _vp(te), _stream_ptr(stream)))

    def factor_stream(self, A_host, R_host, bufs):
        """Host-to-host factorization with every transfer overlapped
        (tqr_qr_host): the arrival units (row chunks of tile columns) of the
        pinned row-major A_host go up in arrival_units() order on one copy
        stream, PACK items consume them as
        they land, UNPACK items write finished R tiles to a device R and a
        second copy stream ships each tile row of R into the pinned R_host
        as soon as it is complete (zeros strictly below the diagonal tiles
        must already be there).  Returns when R_host is filled."""
        assert self.io == (self.IO_IN | self.IO_OUT)
        if not (A_host.is_pinned() and R_host.is_pinned()):
            raise ValueError("A_host and R_host must be page-locked (pin_memory())")
        if A_host.shape != (self.m, self.n) or R_host.shape != (self.n, self.n):
            raise ValueError(f"need A_host {self.m}x{self.n} and R_host {self.n}x{self.n}")
        for name, t in (("A_host", A_host), ("R_host", R_host)):
            if t.dtype != torch.float64 or t.stride(1) != 1 or t.stride(0) < t.shape[1]:
                raise ValueError(f"{name} must be fp64 row-major with unit column stride")
        cs = torch.cuda.current_stream()
        check(lib().tqr_qr_host(self._h, C.c_void_p(A_host.data_ptr()), A_host.stride(0),
                                C.c_void_p(R_host.data_ptr()), R_host.stride(0), _vp(bufs.stage), _vp(bufs.arrive),
                                _vp(bufs.tiles), _vp(bufs.tg), _vp(bufs.te), _vp(bufs.r_dev), _vp(bufs.r_ready),
                                _stream_ptr(cs), _stream_ptr(bufs.copy_in), _stream_ptr(bufs.copy_out)))
        cs.synchronize()

    def stream_buffers(self, device=None):
        """Device scratch for factor_stream (reusable across calls)."""
        dev = device or torch.device("cuda", torch.cuda.current_device())
        tiles, tg, te = self.alloc(dev)
        return StreamBuffers(tiles, tg, te, torch.empty((self.m, self.n), dtype=torch.float64, device=dev),
                             torch.zeros(len(self.arrival_units()), dtype=torch.int32, device=dev),
                             torch.empty((self.n, self.n), dtype=torch.float64, device=dev),
                             torch.zeros(self.q, dtype=torch.int32, device=dev),
                             torch.cuda.Stream(dev), torch.cuda.Stream(dev))

    def arrival_units(self):
        """Input arrival units in host transfer order (tqr_plan_arrival_units):
        (tile column j, first tile row i0, tile rows), 1-based."""
        import numpy as np
        n = C.c_int32()
        check(lib().tqr_plan_arrival_units(self._h, C.byref(n), None))
        out = np.empty(3 * n.value, dtype=np.int32)
        check(lib().tqr_plan_arrival_units(self._h, C.byref(n), _lib.ptr_i32(out)))
        return [tuple(int(v) for v in out[3 * u:3 * u + 3]) for u in range(n.value)]

    def factor_traced(self, tiles, tg, te, stream=None):
        """factor() with a per-work-item device timeline (globaltimer stamps
        at dequeue, dependencies-ready and end, plus the SM id) — returns a
        DeviceTimeline.  The stamps cost a few store instructions per item."""
        import numpy as np
        n = self.info.n_items
        tr = torch.zeros(4 * n + 64, dtype=torch.int64, device=tiles.device)
        check(lib().tqr_set_trace(_vp(tr)))
        try:
            self.factor(tiles, tg, te, stream)
            (stream or torch.cuda.current_stream()).synchronize()
        finally:
            lib().tqr_set_trace(None)
        items = np.empty((n, 7), dtype=np.int32)
        check(lib().tqr_plan_items(self._h, _lib.ptr_i32(items)))
        return DeviceTimeline(items, tr[:4 * n].view(n, 4).cpu().numpy())

    def apply_q(self, trans, tiles, tg, te, c_tiles, c_cols, stream=None):
        check(lib().tqr_apply_q(self._h, int(bool(trans)), _vp(tiles), _vp(tg), _vp(te), _vp(c_tiles),
                                int(c_cols), _stream_ptr(stream)))

    def extract_r(self, tiles, stream=None):
        R = torch.empty((self.n, self.n), dtype=torch.float64, device=tiles.device)
        check(lib().tqr_extract_r(_vp(tiles), self.p, self.q, self.nb, _vp(R), self.n, 1, _stream_ptr(stream)))
        return R

    def unpack(self, tiles, cols=None, stream=None):
        cols = self.q if cols is None else cols
        A = torch.empty((self.m, cols * self.nb), dtype=torch.float64, device=tiles.device)
        check(lib().tqr_unpack(_vp(tiles), self.p, cols, self.nb, _vp(A), A.stride(0), 1, _stream_ptr(stream)))
        return A

    def pack_cols(self, A, cols, stream=None):
        tiles = torch.empty(self.p * cols * self.nb * self.nb, dtype=torch.float64, device=A.device)
        A = A.contiguous()
        check(lib().tqr_pack(_vp(A), A.stride(0), 1, _vp(tiles), self.p, cols, self.nb, _stream_ptr(stream)))
        return tiles


_KIND = ("GEQRT", "TTQRT", "TSQRT", "UNMQR", "TTMQR", "TSMQR", "PACK", "UNPACK")


class DeviceTimeline:
    """Per-work-item timeline of one executor run: item (kind, slab, i, piv,
    k, j) ran on SM `sm` from `start` (its dependencies satisfied) to `end`,
    microseconds from the first dequeue."""

    def __init__(self, items, stamps):
        t0 = stamps[:, 0].min() if len(stamps) else 0
        self.items = items
        self.dequeue = (stamps[:, 0] - t0) / 1e3
        self.start = (stamps[:, 1] - t0) / 1e3
        self.end = (stamps[:, 2] - t0) / 1e3
        self.sm = stamps[:, 3].astype(int)

    @staticmethod
    def _indices(row):
        kind, _, i, piv, k, j = (int(x) for x in row[:6])
        name = _KIND[kind]
        if name == "GEQRT":
            return name, (i, k)
        if name == "UNMQR":
            return name, (i, k, j)
        if name in ("TTQRT", "TSQRT"):
            return name, (i, piv, k)
        if name in ("PACK", "UNPACK"):
            return name, (i, j)
        return name, (i, piv, k, j)

    def gantt_rows(self):
        """(proc, start, end, kind, i, j, k) rows — the layout of the
        reference's Schedule.gantt_rows (sched.py:36-43): the first three
        task indices, padded with "", sorted by (proc, start, kind); proc is
        the SM, times are in microseconds."""
        rows = []
        for r in range(len(self.items)):
            name, idx = self._indices(self.items[r])
            idx = list(idx) + [""] * (3 - len(idx))
            rows.append((int(self.sm[r]), round(float(self.start[r]), 3), round(float(self.end[r]), 3), name,
                         *idx[:3]))
        rows.sort(key=lambda x: (x[0], x[1], x[3]))
        return rows

    def to_csv(self):
        """Gantt CSV, header proc,start,end,kind,i,j,k (sched.py:45-49)."""
        lines = ["proc,start,end,kind,i,j,k"]
        lines += [",".join(str(x) for x in row) for row in self.gantt_rows()]
        return "\n".join(lines) + "\n"

    def makespan_us(self):
        return float(self.end.max()) if len(self.end) else 0.0


@dataclasses.dataclass
class StreamBuffers:
    tiles: torch.Tensor
    tg: torch.Tensor
    te: torch.Tensor
    stage: torch.Tensor
    arrive: torch.Tensor
    r_dev: torch.Tensor
    r_ready: torch.Tensor
    copy_in: torch.cuda.Stream
    copy_out: torch.cuda.Stream


class TiledQR:
    """Result of a tiled QR: factored tiles (R + reflectors) and T factors.
    `shape` is the caller's m x n when the matrix was zero-padded to whole
    tiles (R, Q and apply_q then answer for the unpadded matrix)."""

    def __init__(self, plan: Plan, tiles, tg, te, shape=None):
        self.plan, self.tiles, self.tg, self.te = plan, tiles, tg, te
        self.shape = tuple(shape) if shape is not None else (plan.m, plan.n)

    @property
    def build(self):
        return self.plan.build

    def R(self):
        n = self.shape[1]
        R = self.plan.extract_r(self.tiles)
        return R if n == self.plan.n else R[:n, :n].contiguous()

    def apply_q(self, C_mat, trans=False):
        """Q @ C (trans=False) or Q^T @ C (trans=True) for an m x c device
        matrix (m the factored matrix's rows; zero-padded to whole tiles
        internally)."""
        P = self.plan
        m, c = C_mat.shape
        assert m == self.shape[0], (C_mat.shape, self.shape)
        cols = -(-c // P.nb)
        if (m, c) != (P.m, cols * P.nb):
            Cp = torch.zeros((P.m, cols * P.nb), dtype=torch.float64, device=C_mat.device)
            Cp[:m, :c] = C_mat
            C_mat = Cp
        ct = P.pack_cols(C_mat, cols)
        P.apply_q(trans, self.tiles, self.tg, self.te, ct, cols)
        out = P.unpack(ct, cols)
        return out if out.shape == (m, c) else out[:m, :c].contiguous()

    def Q(self):
        """Explicit m x n Q (reverse reflector replay on [I; 0])."""
        m, n = self.shape
        E = torch.zeros((m, n), dtype=torch.float64, device=self.tiles.device)
        E[:n].fill_diagonal_(1.0)
        return self.apply_q(E, trans=False)


_PLAN_CACHE = {}
_PLAN_CACHE_MAX = 8


def cached_plan(p, q, nb, ib=32, algo="greedy", family="TT", bs=None, grasap_i=1, io=0):
    """Compiled Plan for a tree on p x q tiles, kept in a small per-process
    cache (least recently used out): repeated tiled_qr calls on one shape
    pay the schedule compile (build_tree + tqr_plan_create) once.  Plans
    are immutable and safe to share (per-launch scratch)."""
    key = (p, q, nb, ib, algo.lower(), family, bs, grasap_i, io, torch.cuda.current_device())
    plan = _PLAN_CACHE.pop(key, None)
    if plan is None:
        plan = Plan(build_tree(p, q, algo, family=family, bs=bs, grasap_i=grasap_i), nb, ib, io=io)
    _PLAN_CACHE[key] = plan
    while len(_PLAN_CACHE) > _PLAN_CACHE_MAX:
        _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))
    return plan


def tiled_qr_host(A_host, R_host=None, nb=256, algo="greedy", family="TT", bs=None, grasap_i=1, plan=None,
                  buffers=None):
    """Host matrix in, host R out, with the transfers overlapped with the
    factorization (PACK/UNPACK work items, tqr_qr_host).  A_host: fp64
    m x n row-major (pinned for full overlap); returns (R_host, TiledQR)."""
    A_host = torch.as_tensor(A_host, dtype=torch.float64)
    m, n = A_host.shape
    if m < n:
        raise ValueError(f"need m >= n (got {m}x{n})")
    p, q = -(-m // nb), -(-n // nb)
    shape = (m, n)
    if (p * nb, q * nb) != (m, n):  # zero-pad to whole tiles (see tiled_qr)
        Ap = torch.zeros((p * nb, q * nb), dtype=torch.float64).pin_memory()
        Ap[:m, :n] = A_host
        A_host = Ap
    elif not (A_host.is_pinned() and A_host.stride(1) == 1 and A_host.stride(0) >= A_host.shape[1]):
        A_host = A_host.contiguous().pin_memory()  # row-major, unit column stride
    if plan is None:
        plan = cached_plan(p, q, nb, algo=algo, family=family, bs=bs, grasap_i=grasap_i, io=Plan.IO_IN | Plan.IO_OUT)
    R_pad = R_host if (R_host is not None and shape[1] == q * nb) else None
    if R_pad is None:
        R_pad = torch.zeros((q * nb, q * nb), dtype=torch.float64).pin_memory()
    if buffers is None:
        buffers = plan.stream_buffers()
    plan.factor_stream(A_host, R_pad, buffers)
    if R_pad is not R_host:
        if R_host is None:
            R_host = R_pad[:n, :n].clone()
        else:
            R_host.copy_(R_pad[:n, :n])
    return R_host, TiledQR(plan, buffers.tiles, buffers.tg, buffers.te, shape)


def tiled_qr(A, nb=256, ib=32, algo="greedy", family="TT", bs=None, grasap_i=1, elim=None, plan=None):
    """Tiled QR of an m x n fp64 matrix, m >= n, as p x q tiles of nb x nb
    (nb in {64, 128, 256}).  A matrix that is not a whole number of tiles is
    zero-padded to p = ceil(m/nb), q = ceil(n/nb) (zero rows below and zero
    columns to the right leave R's leading n x n block and Q's leading m x n
    block unchanged: the reflectors never touch zero rows, and zero columns
    give tau = 0).

    The elimination tree is ``build_tree(p, q, algo, family, bs, grasap_i)``
    or the given elimination list ``elim`` (this package's or the
    reference's; validated, tiled_build).  A on the host is copied to the
    current device.  Returns a TiledQR.
    """
    if not torch.cuda.is_available():
        raise RuntimeError("tiled QR needs a CUDA device (no CPU fallback)")
    A = torch.as_tensor(A, dtype=torch.float64)
    m, n = A.shape
    if m < n:
        raise ValueError(f"need m >= n (got {m}x{n})")
    p, q = -(-m // nb), -(-n // nb)
    shape = (m, n)
    if (p * nb, q * nb) != (m, n):
        Ap = torch.zeros((p * nb, q * nb), dtype=torch.float64, device=A.device)
        Ap[:m, :n] = A
        A = Ap
    if plan is None:
        if elim is not None:
            if not (hasattr(elim, "p") and hasattr(elim, "q") and hasattr(elim, "__iter__")):
                raise TypeError("elim must be an elimination list (.p .q and entries .i .piv .k)")
            if (elim.p, elim.q) != (p, q):
                raise ValueError(f"list is for {elim.p}x{elim.q} tiles, matrix has {p}x{q}")
            build = tiled_build(elim, family)
            plan = Plan(build, nb, ib)
        else:
            plan = cached_plan(p, q, nb, ib, algo=algo, family=family, bs=bs, grasap_i=grasap_i)
    if not A.is_cuda:
        A = A.cuda()
    tiles, tg, te = plan.alloc(A.device)
    plan.pack(A, tiles)
    plan.factor(tiles, tg, te)
    return TiledQR(plan, tiles, tg, te, shape)
