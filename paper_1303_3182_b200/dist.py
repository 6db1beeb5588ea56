"""Tall-skinny tiled QR across GPUs (BASELINE config 5).

Block-row partition: rank r owns tile rows [r*P+1, (r+1)*P] of a p x q tile
matrix (P = p/G).  Each rank factors its shard with the reference's Greedy
tree (coarse_schedule, qr.py:254-297) — no communication.  Then log2(G)
rounds of binary TT merges: in round s (stride 2^s) rank b = a + stride
sends the upper block triangle of its q x q-tile R factor to rank a (one
NCCL point-to-point message of q(q+1)/2 tiles), and rank a eliminates the stacked [R_a; R_b] column by column
with TTQRT / TTMQR / GEQRT / UNMQR, pairing rows as soon as they are ready
under the device cost model (the Asap event rule, qr.py:551-583; the
round-1 Greedy-style pairing is kept as merge_pairs_greedy — its critical
path is 1.8x longer).  Written as one global elimination list, local trees plus
merges form a valid list under the reference's validate() (qr.py:56-83)
with unchanged total weight (tests/test_dist.py).

The numerics go through the same engine as the single-GPU path; the
exchange is torch.distributed (NCCL on GPUs).  `Backend` isolates the
device work so the control flow is testable with gloo on CPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .qr import ElimEntry, EliminationList, coarse_schedule
from .taskgraph import GEQRT, QR_KINDS, TTMQR, TTQRT, UNMQR

KIND_ID = {k: n for n, k in enumerate(QR_KINDS)}


# ---------------------------------------------------------------------------
# schedule side (host, exact)

# device cost model of the merge pairing (units of ~30 us at nb=256, measured
# in the executor: TTQRT ~ GEQRT ~ 450 us, one TTMQR tile update ~ 60 us with
# its four 64-column slabs in parallel)
MERGE_COST = {"ttqrt": 15, "ttmqr": 2, "geqrt": 15}


def merge_pairs_greedy(q, row_a, rows_b):
    """Greedy-style pairing (round-1 merges, kept for comparison): per column
    k the live rows are [row_a(k)] + [rows_b(i) for i <= k]; while more than
    one is live, the bottom z = len//2 are zeroed by the z rows directly
    above them.  Simulated critical path at q = 8:
    13.0 ms vs 7.2 ms for merge_pairs."""
    out = []
    for k in range(1, q + 1):
        live = [row_a(k)] + [rows_b(i) for i in range(1, k + 1)]
        while len(live) > 1:
            z = len(live) // 2
            tg, pv = live[len(live) - z:], live[len(live) - 2 * z:len(live) - z]
            for t, v in zip(tg, pv):
                out.append(ElimEntry(t, v, k))
            live = live[:len(live) - z]
    return out


def merge_pairs_multi(q, rows_of, cost=None):
    """Eliminations merging G upper block-triangular R factors (block g's
    row i is rows_of[g](i); block 0 holds the result), paired as soon as
    possible (the event rule of the reference's Asap, qr.py:551-583, under
    the device cost model): per column k the live rows are row k of every
    block (ready at once: untouched by earlier columns) and the rows
    eliminated in column k-1 (ready after their TTMQR on column k and the
    GEQRT that re-triangularizes it).  The two earliest-ready rows pair, the
    lower merge row (block 0's row k when involved: it ends as R's row k)
    survives and is ready again after the TTQRT.  Entries are emitted in
    simulated start order (ties: row numbers), a valid list order."""
    import heapq

    c = cost or MERGE_COST
    G = len(rows_of)
    ev, carry = [], []
    for k in range(1, q + 1):
        live = [(0, g * q + k) for g in range(G)] + carry  # (ready time, merge row)
        carry = []
        heapq.heapify(live)
        while len(live) > 1:
            t1, r1 = heapq.heappop(live)
            t2, r2 = heapq.heappop(live)
            s = max(t1, t2)
            piv, tgt = (r1, r2) if r1 < r2 else (r2, r1)
            ev.append((s, tgt, piv, k))
            heapq.heappush(live, (s + c["ttqrt"], piv))
            carry.append((s + c["ttqrt"] + c["ttmqr"] + c["geqrt"], tgt))
        assert live[0][1] == k
    ev.sort()
    row = lambda r: rows_of[(r - 1) // q]((r - 1) % q + 1)  # noqa: E731
    return [ElimEntry(row(t), row(v), k) for _, t, v, k in ev]


def merge_pairs(q, row_a, rows_b, cost=None):
    """Two-block merge_pairs_multi: R_a (rows row_a(k)) with R_b."""
    return merge_pairs_multi(q, [row_a, rows_b], cost)


def composite_list(p, q, G, merge="binary"):
    """Global elimination list of G local Greedy trees + the merges:
    log2 G rounds of binary merges (merge="binary", SURVEY.md App. B.2 with
    Asap pairing) or one gather merge of all G R factors on block 0
    (merge="gather")."""
    if p % G:
        raise ValueError("p must be a multiple of the number of shards")
    P = p // G
    if P < q:
        raise ValueError("each shard needs at least q tile rows")
    _, local = coarse_schedule(P, q, "greedy")
    entries = []
    for s in range(G):
        entries += [ElimEntry(e.i + s * P, e.piv + s * P, e.k) for e in local]
    if merge == "gather":
        if G > 1:
            entries += merge_pairs_multi(q, [lambda i, g=g: g * P + i for g in range(G)])
        return EliminationList(p, q, entries).with_steps()
    stride = 1
    while stride < G:
        for a in range(0, G, 2 * stride):
            b = a + stride
            if b < G:
                entries += merge_pairs(q, lambda k, a=a: a * P + k, lambda i, b=b: b * P + i)
        stride *= 2
    return EliminationList(p, q, entries).with_steps()


def merge_trace(q, G=2):
    """Kernel trace of one merge on the stacked G q x q tile matrix
    [R_0; R_1; ...] (rows g q + 1 .. g q + q = R_g): the TT bundle of each
    merge elimination (qr.py:494-502) — TTQRT, TTMQR for j > k, and the
    eliminated row re-triangularized in column k+1 (GEQRT + UNMQR).  Tiles
    below the block diagonals are structurally zero and never touched."""
    kinds, idx = [], []
    for e in merge_pairs_multi(q, [lambda i, g=g: g * q + i for g in range(G)]):
        kinds.append(KIND_ID[TTQRT])
        idx.append((e.i, e.piv, e.k, -1))
        for j in range(e.k + 1, q + 1):
            kinds.append(KIND_ID[TTMQR])
            idx.append((e.i, e.piv, e.k, j))
        if e.k + 1 <= q:
            kinds.append(KIND_ID[GEQRT])
            idx.append((e.i, e.k + 1, -1, -1))
            for j in range(e.k + 2, q + 1):
                kinds.append(KIND_ID[UNMQR])
                idx.append((e.i, e.k + 1, j, -1))
    return np.asarray(kinds, dtype=np.int8), np.asarray(idx, dtype=np.int32).reshape(-1, 4)


def emulate(A, G, nb, backend_cls=None, device=None, keep=False, merge="binary"):
    """Single-device emulation of tall_skinny_qr with G shards (same local
    trees and merge order; the exchange is a device copy).  For tests.
    keep=True gives every shard its own backend (the local factors stay for
    emulate_apply_q) and returns the list of backends."""
    p, q = A.shape[0] // nb, A.shape[1] // nb
    P = p // G
    cls = backend_cls or GpuBackend
    bes = [cls(P, q, nb, device) for _ in range(G)] if keep else [cls(P, q, nb, device)] * G
    rs = []
    for s in range(G):
        rs.append(bes[s].factor_local(A[s * P * nb:(s + 1) * P * nb]).clone())
    if merge == "gather":
        if G > 1:
            rs[0] = bes[0].merge_many(rs, key="gather" if keep else None).clone()
        return (bes if keep else bes[0]), rs[0]
    for stride, pairs in merge_rounds(G):
        for a, b in pairs:
            m = bes[a].merge(rs[a], rs[b], key=stride) if keep else bes[a].merge(rs[a], rs[b])
            rs[a] = m.clone()
    return (bes if keep else bes[0]), rs[0]


def emulate_apply_q(bes, C, trans, merge="binary"):
    """Q^T C (trans) or Q C of an emulate(..., keep=True) factorization; C is
    the global m x c device matrix, split by the same block rows."""
    G = len(bes)
    P, q, nb = bes[0].P, bes[0].q, bes[0].nb
    cs = [C[s * P * nb:(s + 1) * P * nb].clone() for s in range(G)]
    h = q * nb
    rounds = merge_rounds(G)
    if trans:
        cs = [be.apply_local(c, True) for be, c in zip(bes, cs)]
    if merge == "gather":
        if G > 1:
            outs = bes[0].apply_merge_many("gather", [c[:h] for c in cs], trans)
            for c, o in zip(cs, outs):
                c[:h].copy_(o)
        rounds = []
    for stride, pairs in (rounds if trans else rounds[::-1]):
        for a, b in pairs:
            ta, tb = bes[a].apply_merge(stride, cs[a][:h], cs[b][:h], trans)
            cs[a][:h].copy_(ta)
            cs[b][:h].copy_(tb)
    if not trans:
        cs = [be.apply_local(c, False) for be, c in zip(bes, cs)]
    return cs


def merge_rounds(G):
    """[(stride, [(a, b), ...]), ...] — who sends (b) to whom (a)."""
    out, stride = [], 1
    while stride < G:
        out.append((stride, [(a, a + stride) for a in range(0, G, 2 * stride) if a + stride < G]))
        stride *= 2
    return out


# ---------------------------------------------------------------------------
# device side

class GpuBackend:
    """Local factorization and merges with the libtqr engine."""

    def __init__(self, P, q, nb, device, algo="greedy", family="TT"):
        import torch

        from .engine import Plan
        from .qr import QrBuild, build_tree

        self.torch = torch
        self.P, self.q, self.nb, self.dev = P, q, nb, device
        self.local_plan = Plan(build_tree(P, q, algo, family=family), nb)
        self.tiles, self.tg, self.te = self.local_plan.alloc(device)
        self._merges = {}  # G stacked R blocks -> (plan, tiles, tg, te)
        self._merge_setup(2)
        t2 = nb * nb
        self.rbuf = torch.empty(q * q * t2, dtype=torch.float64, device=device)
        self.merge_factors = {}  # merge key (round stride) -> (tiles, tg, te)

    def factor_local(self, A_local):
        self.local_plan.pack(A_local, self.tiles)
        self.local_plan.factor(self.tiles, self.tg, self.te)
        # R tile rows 1..q of every tile column -> (q cols) x (q tiles)
        t2 = self.nb * self.nb
        src = self.tiles.view(self.q, self.P * t2)[:, :self.q * t2]
        self.rbuf.view(self.q, self.q * t2).copy_(src)
        return self.rbuf

    def factor_local_host(self, A_host):
        """factor_local from a page-locked host shard: the column blocks
        stream in on a copy stream while the executor factors (PACK items,
        tqr_qr_host with io=1)."""
        torch = self.torch
        if getattr(self, "io_plan", None) is None:
            from .engine import Plan
            self.io_plan = Plan(self.local_plan.build, self.nb, io=Plan.IO_IN)
            self.stage = torch.empty((self.P * self.nb, self.q * self.nb), dtype=torch.float64, device=self.dev)
            self.arrive = torch.zeros(len(self.io_plan.arrival_units()), dtype=torch.int32, device=self.dev)
            self.copy_in = torch.cuda.Stream(self.dev)
        cs = torch.cuda.current_stream()
        vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        _lib.check(_lib.lib().tqr_qr_host(self.io_plan._h, C.c_void_p(A_host.data_ptr()), A_host.stride(0), None, 0,
                                          vp(self.stage), vp(self.arrive), vp(self.tiles), vp(self.tg), vp(self.te),
                                          None, None, C.c_void_p(cs.cuda_stream),
                                          C.c_void_p(self.copy_in.cuda_stream), C.c_void_p(self.copy_in.cuda_stream)))
        t2 = self.nb * self.nb
        src = self.tiles.view(self.q, self.P * t2)[:, :self.q * t2]
        self.rbuf.view(self.q, self.q * t2).copy_(src)
        return self.rbuf

    def _merge_setup(self, G):
        """Plan + buffers of the merge of G stacked R blocks (merge_trace)."""
        if G not in self._merges:
            from .engine import Plan
            from .qr import QrBuild
            kinds, idx = merge_trace(self.q, G)
            h = C.c_void_p()
            _lib.check(_lib.lib().tqr_trace_build(G * self.q, self.q, kinds.ctypes.data_as(_lib.i8p),
                                                  _lib.ptr_i32(idx), len(kinds), C.byref(h)))
            mb = QrBuild.__new__(QrBuild)
            mb.__dict__.update(p=G * self.q, q=self.q, family="TT", keep_trace=True, _h=h, record_updates=False)
            plan = Plan(mb, self.nb)
            self._merges[G] = (plan, *plan.alloc(self.dev))
        return self._merges[G]

    def merge_many(self, rs, key=None):
        """[R_0; R_1; ...; R_{G-1}] -> merged R (q x q tiles, written into
        rs[0]), one executor launch (merge_trace(q, G)).  With a key the
        merge's reflectors and T factors are kept for apply_merge_many."""
        G, q, t2 = len(rs), self.q, self.nb * self.nb
        plan, tiles, tg, te = self._merge_setup(G)
        m = tiles.view(q, G * q * t2)
        for g, r in enumerate(rs):
            m[:, g * q * t2:(g + 1) * q * t2].copy_(r.view(q, q * t2))
        plan.factor(tiles, tg, te)
        if key is not None:
            self.merge_factors[key] = (G, tiles.clone(), tg.clone(), te.clone())
        rs[0].view(q, q * t2).copy_(m[:, :q * t2])
        return rs[0]

    def merge(self, r_a, r_b, key=None):
        """[R_a; R_b] -> merged R (q x q tiles, written into r_a); see
        merge_many."""
        return self.merge_many([r_a, r_b], key)

    def apply_local(self, C, trans):
        """Q_local^T C (trans) or Q_local C for this shard's block rows
        C (P*nb x c, device); the local factors of the last factor_local."""
        plan = self.local_plan
        cols = C.shape[1] // self.nb
        ct = plan.pack_cols(C, cols)
        plan.apply_q(trans, self.tiles, self.tg, self.te, ct, cols)
        return plan.unpack(ct, cols)

    def apply_merge_many(self, key, tops, trans):
        """The merge `key`'s Q^T (trans) or Q applied to the stacked R-rows
        [tops[0]; tops[1]; ...] of C (q*nb x c each); returns the pieces."""
        G, tiles, tg, te = self.merge_factors[key]
        plan, h = self._merge_setup(G)[0], self.q * self.nb
        cols = tops[0].shape[1] // self.nb
        ct = plan.pack_cols(self.torch.cat(tops), cols)
        plan.apply_q(trans, tiles, tg, te, ct, cols)
        out = plan.unpack(ct, cols)
        return [out[g * h:(g + 1) * h] for g in range(G)]

    def apply_merge(self, key, top_a, top_b, trans):
        """Two-block apply_merge_many; returns the two halves."""
        return tuple(self.apply_merge_many(key, [top_a, top_b], trans))

    def r_matrix(self, rbuf):
        """Upper-triangular n x n R from a q x q tile block."""
        R = self.torch.empty((self.q * self.nb, self.q * self.nb), dtype=self.torch.float64, device=self.dev)
        _lib.check(_lib.lib().tqr_extract_r(C.c_void_p(rbuf.data_ptr()), self.q, self.q, self.nb,
                                            C.c_void_p(R.data_ptr()), R.shape[1], 1,
                                            C.c_void_p(self.torch.cuda.current_stream().cuda_stream)))
        return R


def _upper_tiles(q):
    """Flat indices of the R tiles (i <= j) in a [q cols][q tiles] block."""
    return [j * q + i for j in range(q) for i in range(j + 1)]


def tall_skinny_qr(A_local, backend, rank, world, dist=None, keep_q=False, merge="binary"):
    """Factor the block rows A_local on every rank; rank 0 returns the final
    q x q-tile R block (others return None).  `dist` is torch.distributed
    (send/recv of the R block; NCCL on GPUs, gloo in the CPU tests).  Only
    the q(q+1)/2 tiles of R's upper block triangle travel (18 MiB at q = 8
    instead of 32): the merge trace never reads a tile below the block
    diagonal.  merge="gather": every rank sends its block to rank 0 at once
    and rank 0 merges all G in one launch (merge_many: one exchange step and
    a critical path of ~1.6 binary merges at G = 8 instead of log2 G = 3).
    A_local on the host (page-locked, GpuBackend) streams in while the local
    factorization runs.  keep_q keeps every merge's factors on the receiving
    rank for tall_skinny_apply_q (the local factors stay in the backend
    until its next factorization)."""
    if getattr(A_local, "is_cuda", True) or not hasattr(backend, "factor_local_host"):
        r = backend.factor_local(A_local)
    else:
        r = backend.factor_local_host(A_local)
    rounds = merge_rounds(world)
    if not rounds:
        return r if rank == 0 else None
    import torch
    q = backend.q
    t2 = r.numel() // (q * q)
    up = torch.tensor(_upper_tiles(q), dtype=torch.long, device=r.device)
    if merge == "gather":
        if rank != 0:
            dist.send(r.view(q * q, t2).index_select(0, up), dst=0)
            return None
        packed = [r.new_empty((len(up), t2)) for _ in range(world - 1)]
        reqs = [dist.irecv(packed[g - 1], src=g) for g in range(1, world)]
        rs = [r]
        for g in range(1, world):
            reqs[g - 1].wait()
            full = r.new_zeros(r.shape)
            full.view(q * q, t2).index_copy_(0, up, packed[g - 1])
            rs.append(full)
        return backend.merge_many(rs, key="gather" if keep_q else None)
    recv = None
    for stride, pairs in rounds:
        for a, b in pairs:
            if rank == b:
                dist.send(r.view(q * q, t2).index_select(0, up), dst=a)
            elif rank == a:
                if recv is None:
                    recv = r.new_zeros(r.shape)
                    packed = r.new_empty((len(up), t2))
                dist.recv(packed, src=b)
                recv.view(q * q, t2).index_copy_(0, up, packed)
                r = backend.merge(r, recv, key=stride) if keep_q else backend.merge(r, recv)
    return r if rank == 0 else None


def tall_skinny_apply_q(C_local, backend, rank, world, trans, dist=None, merge="binary"):
    """Q^T C (trans=True) or Q C (trans=False) for the Q of a
    tall_skinny_qr(..., keep_q=True) on the same ranks: C is block-row
    sharded like A (C_local: this rank's P*nb rows, on the backend's device).
    Q = Q_local(r) . merges in round order, so Q^T applies every rank's local
    reflectors, then each round's merge to the stacked R-rows (the first
    q*nb rows of each shard) on the receiving rank — the sender's rows go
    there and come back (point-to-point, like the R exchange); Q applies
    them in reverse.  Returns this rank's rows of the result."""
    h = backend.q * backend.nb
    rounds = merge_rounds(world)
    c = backend.apply_local(C_local, True) if trans else C_local.clone()
    if merge == "gather" and world > 1:
        # the stacked R-rows of every rank go to rank 0 and come back
        if rank != 0:
            top = c[:h].contiguous()
            dist.send(top, dst=0)
            dist.recv(top, src=0)
            c[:h].copy_(top)
        else:
            tops = [c[:h]] + [c[:h].new_empty(c[:h].shape) for _ in range(world - 1)]
            for g in range(1, world):
                dist.recv(tops[g], src=g)
            outs = backend.apply_merge_many("gather", tops, trans)
            c[:h].copy_(outs[0])
            for g in range(1, world):
                dist.send(outs[g].contiguous(), dst=g)
        rounds = []
    for stride, pairs in (rounds if trans else rounds[::-1]):
        for a, b in pairs:
            if rank == b:
                top = c[:h].contiguous()
                dist.send(top, dst=a)
                dist.recv(top, src=a)
                c[:h].copy_(top)
            elif rank == a:
                tb = c[:h].new_empty(c[:h].shape)
                dist.recv(tb, src=b)
                ta, tb = backend.apply_merge(stride, c[:h], tb, trans)
                c[:h].copy_(ta)
                dist.send(tb.contiguous(), dst=b)
    if not trans:
        c = backend.apply_local(c, False)
    return c
