"""Tall-skinny multi-GPU path: schedule facts on CPU, the
NCCL exchange pattern exercised with gloo (world_size 2) and the LAPACK
replay oracle standing in for the device kernels, and (GPU) the device
merges emulated on one GPU."""
import os
import socket

import numpy as np
import pytest
import torch

import paper_1303_3182_b200 as P
from paper_1303_3182_b200 import dist
from oracle.replay import Replay, replay_build, row_sign_normalize

from _digest import build_digest, elim_sha


@pytest.mark.parametrize("key", ["64/8/8", "16/4/2", "16/4/4", "8192/8/1", "8192/8/2", "8192/8/8"])
def test_composite_list_matches_reference(golden, key):
    p, q, G = (int(x) for x in key.split("/"))
    rec = golden["composite"][key]
    lst = dist.composite_list(p, q, G)
    assert lst.validate()
    assert len(lst) == rec["nelim"] and elim_sha(lst) == rec["elim_sha"]
    b = P.tiled_build(lst, keep_trace=(p <= 64))
    assert b.cp == rec["cp"] and b.total_weight == rec["total_weight"] == P.total_weight(p, q)
    if "trace_sha" in rec:
        assert build_digest(b) == rec["trace_sha"]


@pytest.mark.parametrize("p,q,G", [(64, 8, 8), (16, 4, 4), (24, 4, 3), (8192, 8, 8)])
def test_gather_composite_list_valid(p, q, G):
    """Local Greedy trees + one gather merge of all G R factors: a valid
    elimination list under the reference's rules (qr.py:56-83, the C++
    validator), total weight unchanged (qr.py:663-677)."""
    lst = dist.composite_list(p, q, G, merge="gather")
    assert lst.validate()
    b = P.tiled_build(lst, keep_trace=False)
    assert b.total_weight == P.total_weight(p, q)
    kinds, _ = dist.merge_trace(q, G)
    assert len(kinds) > 0


def test_merge_trace_is_the_tail_of_the_global_trace():
    p, q, G = 16, 4, 2
    Pp = p // G
    b = P.tiled_build(dist.composite_list(p, q, G))
    kinds, idx, _ = b.trace_arrays()
    mk, mi = dist.merge_trace(q)
    tail_k, tail_i = kinds[-len(mk):], idx[-len(mk):]
    assert (tail_k == mk).all()

    def to_local(r):  # global row -> merge-matrix row
        if r <= 0:
            return r
        return r if r <= Pp else q + (r - Pp)
    arity = (2, 3, 3, 3, 4, 4)
    for kd, g, l in zip(tail_k, tail_i, mi):
        n_rows = 1 if kd in (0, 3) else 2
        exp = [to_local(int(x)) if t < n_rows else int(x) for t, x in enumerate(g[:arity[kd]])]
        assert exp == [int(x) for x in l[:arity[kd]]]


class CpuOracleBackend:
    """LAPACK-replay stand-in for GpuBackend (test infrastructure only)."""

    def __init__(self, Pp, q, nb, device=None):
        self.Pp, self.q, self.nb = Pp, q, nb

    def _block(self, tiles):
        out = torch.empty(self.q * self.q * self.nb * self.nb, dtype=torch.float64)
        v = out.view(self.q, self.q, self.nb * self.nb)
        for j in range(self.q):
            for i in range(self.q):
                v[j, i] = torch.from_numpy(np.ascontiguousarray(tiles[i][j].reshape(-1, order="F")))
        return out

    def _tiles(self, blk):
        v = blk.view(self.q, self.q, self.nb * self.nb).numpy()
        return [[np.asfortranarray(v[j, i].reshape(self.nb, self.nb, order="F")) for j in range(self.q)]
                for i in range(self.q)]

    def factor_local(self, A_local):
        b = P.build_tree(self.Pp, self.q, "greedy")
        rp = replay_build(A_local.numpy(), b, self.nb)
        self.local = (rp, *b.trace_arrays()[:2])
        self.merges = {}
        return self._block(rp.t)

    def merge_many(self, rs, key=None):
        G = len(rs)
        kinds, idx = dist.merge_trace(self.q, G)
        rp = Replay.__new__(Replay)
        rp.p, rp.q, rp.nb, rp.ib = G * self.q, self.q, self.nb, 32
        rp.t = sum((self._tiles(r) for r in rs), [])
        rp.tg, rp.te = {}, {}
        rp.run(kinds, idx)
        if key is not None:
            self.merges[key] = (rp, kinds, idx)
        return self._block(rp.t[:self.q])

    def merge(self, r_a, r_b, key=None):
        return self.merge_many([r_a, r_b], key)

    def apply_local(self, C, trans):
        return torch.from_numpy(_replay_apply(*self.local, C.numpy(), trans))

    def apply_merge_many(self, key, tops, trans):
        out = _replay_apply(*self.merges[key], np.vstack([t.numpy() for t in tops]), trans)
        h = self.q * self.nb
        return [torch.from_numpy(out[g * h:(g + 1) * h].copy()) for g in range(len(tops))]

    def apply_merge(self, key, top_a, top_b, trans):
        return tuple(self.apply_merge_many(key, [top_a, top_b], trans))


def _replay_apply(rp, kinds, idx, C, trans):
    """LAPACK (dgemqrt / dtpmqrt) application of a replayed factorization's
    Q^T (trace order, trans='T') or Q (reverse order, 'N') to C."""
    from scipy.linalg import lapack as L
    nb, p = rp.nb, rp.p
    ct = [np.asfortranarray(C[i * nb:(i + 1) * nb]) for i in range(p)]
    order = range(len(kinds)) if trans else range(len(kinds) - 1, -1, -1)
    tr = "T" if trans else "N"
    for t in order:
        kd = int(kinds[t])
        a, b, c, _ = (int(x) - 1 for x in idx[t])
        if kd == 0:  # GEQRT(a, b)
            ct[a], info = L.dgemqrt(rp.t[a][b], rp.tg[(a, b)], ct[a], side="L", trans=tr)
        elif kd in (1, 2):  # TTQRT / TSQRT(a, piv=b, k=c)
            l = nb if kd == 1 else 0
            v = np.triu(rp.t[a][c]) if l else rp.t[a][c]
            ct[b], ct[a], info = L.dtpmqrt(l, v, rp.te[(a, c)], ct[b], ct[a], side="L", trans=tr)
        else:
            continue
        assert info == 0
    return np.vstack(ct)


def _full_r(blk, q, nb):
    v = blk.view(q, q, nb * nb).numpy()
    R = np.zeros((q * nb, q * nb))
    for j in range(q):
        for i in range(j + 1):
            R[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb] = v[j, i].reshape(nb, nb, order="F")
    return np.triu(R)


def _matrix(p, q, nb, seed=4):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (p * nb, q * nb))


def _worker(rank, world, port, p, q, nb, out, merge="binary"):
    import torch.distributed as td
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    A = _matrix(p, q, nb)
    Pp = p // world
    A_local = torch.from_numpy(A[rank * Pp * nb:(rank + 1) * Pp * nb].copy())
    be = CpuOracleBackend(Pp, q, nb)
    r = dist.tall_skinny_qr(A_local, be, rank, world, td, keep_q=True, merge=merge)
    # distributed apply-Q: Q^T A = [R; 0] on the block rows, Q [I; 0] = Q
    qta = dist.tall_skinny_apply_q(A_local.clone(), be, rank, world, True, td, merge=merge)
    E = np.zeros_like(A)
    E[:q * nb] = np.eye(q * nb)
    ql = dist.tall_skinny_apply_q(torch.from_numpy(E[rank * Pp * nb:(rank + 1) * Pp * nb].copy()), be, rank, world,
                                  False, td, merge=merge)
    parts = [torch.empty_like(ql) for _ in range(world)]
    td.all_gather(parts, ql)
    tparts = [torch.empty_like(qta) for _ in range(world)]
    td.all_gather(tparts, qta)
    if rank == 0:
        Rf = _full_r(r, q, nb)
        R = row_sign_normalize(Rf)
        Rref = row_sign_normalize(np.linalg.qr(A, mode="r"))
        Q = torch.cat(parts).numpy()
        QtA = torch.cat(tparts).numpy()
        nA = np.linalg.norm(A)
        out.put((float(np.linalg.norm(R - Rref) / nA), float(np.linalg.norm(A - Q @ Rf) / nA),
                 float(np.linalg.norm(Q.T @ Q - np.eye(q * nb))),
                 float(np.linalg.norm(QtA - np.vstack([Rf, np.zeros((A.shape[0] - q * nb, q * nb))])) / nA)))
    td.destroy_process_group()


@pytest.mark.parametrize("world,merge", [(2, "binary"), (4, "binary"), (4, "gather"), (3, "gather")])
def test_gloo_exchange_and_merge(world, merge):
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, port, 4 * world, 2, 64, q, merge), nprocs=world, join=True)
    err_r, res, orth, qta = q.get(timeout=60)
    assert err_r <= 1e-13, err_r
    assert res <= 1e-14 and orth <= 1e-13 and qta <= 1e-14, (res, orth, qta)


@pytest.mark.gpu
@pytest.mark.parametrize("G,p,q,nb,merge", [(2, 8, 2, 64, "binary"), (4, 16, 4, 64, "binary"), (2, 8, 4, 256, "binary"),
                                            (4, 16, 4, 64, "gather"), (8, 32, 4, 256, "gather")])
def test_gpu_emulated_shards(G, p, q, nb, merge):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    A = _matrix(p, q, nb, seed=7)
    At = torch.from_numpy(A).cuda()
    be, r = dist.emulate(At, G, nb, device=torch.device("cuda"), merge=merge)
    R = row_sign_normalize(be.r_matrix(r).cpu().numpy())
    Rref = row_sign_normalize(np.linalg.qr(A, mode="r"))
    assert np.linalg.norm(R - Rref) <= 1e-11 * np.linalg.norm(A)


@pytest.mark.gpu
def test_gpu_streamed_local_factorization_matches_device_path():
    """GpuBackend.factor_local_host (page-locked host shard streamed in with
    PACK items) gives the same R block as factor_local on a device copy."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    P, q, nb = 16, 4, 64
    A = _matrix(P, q, nb, seed=11)
    be = dist.GpuBackend(P, q, nb, torch.device("cuda"))
    r_dev = be.factor_local(torch.from_numpy(A).cuda()).clone()
    r_host = be.factor_local_host(torch.from_numpy(A).pin_memory()).clone()
    torch.cuda.synchronize()
    assert torch.equal(r_dev, r_host)


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["TT", "TS"])
def test_gpu_backend_local_family(family):
    """GpuBackend's local tree in either kernel family (tiledag family= of
    build_tree; TS: lazily triangularized pivots, TSQRT/TSMQR for rows that
    never were pivots): the same R up to row signs."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    P, q, nb = 16, 4, 64
    A = _matrix(P, q, nb, seed=17)
    be = dist.GpuBackend(P, q, nb, torch.device("cuda"), family=family)
    assert be.local_plan.build.family == family
    rb = be.factor_local(torch.from_numpy(A).cuda())
    R = row_sign_normalize(be.r_matrix(rb).cpu().numpy())
    Rref = row_sign_normalize(np.linalg.qr(A, mode="r"))
    assert np.linalg.norm(R - Rref) <= 1e-11 * np.linalg.norm(A)


@pytest.mark.gpu
@pytest.mark.parametrize("G,p,q,nb,merge", [(2, 8, 2, 64, "binary"), (4, 16, 4, 64, "binary"), (4, 16, 2, 256, "binary"),
                                            (4, 16, 4, 64, "gather"), (8, 16, 2, 256, "gather")])
def test_gpu_emulated_apply_q(G, p, q, nb, merge):
    """Distributed apply-Q on the device (shards emulated on one GPU):
    Q [I; 0] is orthonormal with A = Q R, and Q^T A = [R; 0]."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    A = _matrix(p, q, nb, seed=13)
    At = torch.from_numpy(A).cuda()
    bes, r = dist.emulate(At, G, nb, device=torch.device("cuda"), keep=True, merge=merge)
    Rf = bes[0].r_matrix(r)
    n = q * nb
    E = torch.zeros_like(At)
    E[:n].fill_diagonal_(1.0)
    Q = torch.cat(dist.emulate_apply_q(bes, E, False, merge=merge))
    QtA = torch.cat(dist.emulate_apply_q(bes, At, True, merge=merge))
    nA = torch.linalg.norm(At)
    assert torch.linalg.norm(At - Q @ Rf) / nA <= 1e-12
    assert torch.linalg.norm(Q.T @ Q - torch.eye(n, dtype=torch.float64, device="cuda")) <= 1e-12
    Z = torch.zeros_like(At)
    Z[:n] = Rf
    assert torch.linalg.norm(QtA - Z) / nA <= 1e-12
