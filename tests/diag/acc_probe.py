"""Accuracy probe: orthogonality of Q from our kernels vs the LAPACK replay
for small tile grids (one GEQRT; one TT elimination; 4x4 tiles)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1303_3182_b200 as P
from paper_1303_3182_b200.engine import tiled_qr
from oracle.replay import replay_build

nb = 256
for (p, q, algo) in [(1, 1, "greedy"), (2, 1, "greedy"), (4, 4, "greedy"), (8, 8, "greedy"), (16, 16, "greedy")]:
    A = np.random.default_rng(2).standard_normal((p * nb, q * nb))
    res = tiled_qr(A, nb=nb, algo=algo)
    Q = res.Q().cpu().numpy()
    R = res.R().cpu().numpy()
    n = q * nb
    o_gpu = np.linalg.norm(Q.T @ Q - np.eye(n))
    r_gpu = np.linalg.norm(A - Q @ R) / np.linalg.norm(A)
    if p * q <= 64:
        b = P.build_tree(p, q, algo)
        rp = replay_build(A, b, nb)
        kinds, idx, _ = b.trace_arrays()
        Qr = rp.form_q(kinds, idx)
        o_ref = np.linalg.norm(Qr.T @ Qr - np.eye(n))
        r_ref = np.linalg.norm(A - Qr @ rp.r()) / np.linalg.norm(A)
        # Q from our factors, formed on the CPU by the replay machinery
        from oracle.replay import Replay
        rq = Replay.__new__(Replay)
        rq.p, rq.q, rq.nb, rq.ib = p, q, nb, 32
        tl = res.tiles.cpu().numpy().reshape(q, p, nb * nb)
        rq.t = [[np.asfortranarray(tl[j, i].reshape(nb, nb, order="F")) for j in range(q)] for i in range(p)]
        tg = res.tg.cpu().numpy().reshape(q, p, 32 * nb)
        te = res.te.cpu().numpy().reshape(q, p, 32 * nb)
        rq.tg = {(i, k): np.asfortranarray(tg[k, i].reshape(32, nb, order="F")) for i in range(p) for k in range(q)}
        rq.te = {(i, k): np.asfortranarray(te[k, i].reshape(32, nb, order="F")) for i in range(p) for k in range(q)}
        Qx = rq.form_q(kinds, idx)
        o_x = np.linalg.norm(Qx.T @ Qx - np.eye(n))
        print(f"{p}x{q}: gpu orth {o_gpu:.2e} resid {r_gpu:.2e} | lapack orth {o_ref:.2e} resid {r_ref:.2e} | our factors, cpu-formed Q orth {o_x:.2e}", flush=True)
    else:
        print(f"{p}x{q}: gpu orth {o_gpu:.2e} resid {r_gpu:.2e}", flush=True)
