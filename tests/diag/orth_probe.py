"""Orthogonality of Q formed from the LAPACK tile replay of the C3 Greedy trace
(reduced n) in fp64 vs 80-bit long double (numpy longdouble), optionally with
T recomputed exactly from V and tau: separates the reflectors' intrinsic
non-orthogonality from the rounding of the Q formation.  CPU only.
Usage: python tools/orth_probe.py N {f64|ld|f64fix|ldfix}"""
import sys, time, numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))))
import paper_1303_3182_b200 as P
from oracle.replay import replay_build
n = int(sys.argv[1]); nb = 256; ib = 32; mode = sys.argv[2]
FORM = np.longdouble if "ld" in mode else np.float64
A = np.random.default_rng(2).standard_normal((n, n))
b = P.build_tree(n // nb, n // nb, "greedy")
rp = replay_build(A, b, nb)
kinds, idx, _ = b.trace_arrays()
def exact_T(V, T):
    # recompute each ib-block T from V and tau (diag) in longdouble (dlarft forward columnwise)
    Tn = np.zeros_like(T)
    VL = V.astype(np.longdouble)
    for blk in range(nb // ib):
        s = slice(blk*ib, (blk+1)*ib); Vb = VL[:, s]; tau = np.diag(T[:, s]).astype(np.longdouble)
        G = Vb.T @ Vb
        Tb = np.zeros((ib, ib), dtype=np.longdouble)
        for j in range(ib):
            Tb[j, j] = tau[j]
            if j: Tb[:j, j] = -tau[j] * (Tb[:j, :j] @ G[:j, j])
        Tn[:, s] = Tb.astype(np.float64)
    return Tn
p = q = n // nb
Q = [[np.zeros((nb, nb), dtype=FORM) for _ in range(q)] for _ in range(p)]
for d in range(q): Q[d][d] = np.eye(nb, dtype=FORM)
fixT = "fix" in mode
for t in range(len(kinds) - 1, -1, -1):
    kd = int(kinds[t]); a, bb, c, _ = (int(x) - 1 for x in idx[t])
    if kd == 0:
        V = np.tril(rp.t[a][bb], -1) + np.eye(nb); T = np.asarray(rp.tg[(a, bb)])
        if fixT: T = exact_T(V, T)
        V = V.astype(FORM); T = T.astype(FORM)
        for blk in range(nb // ib - 1, -1, -1):
            s = slice(blk*ib, (blk+1)*ib); Vb = V[:, s]; Tb = T[:, s]
            for j in range(q):
                C = Q[a][j]; Q[a][j] = C - Vb @ (Tb @ (Vb.T @ C))
    elif kd == 1:
        i, piv, k = a, bb, c
        VE = np.triu(rp.t[i][k]); T = np.asarray(rp.te[(i, k)])
        if fixT:
            T = exact_T(np.vstack([np.eye(nb), VE]), T)
        VE = VE.astype(FORM); T = T.astype(FORM)
        for blk in range(nb // ib - 1, -1, -1):
            s = slice(blk*ib, (blk+1)*ib); Vb = VE[:, s]; Tb = T[:, s]
            for j in range(q):
                Cp = Q[piv][j].copy(); Ci = Q[i][j]
                W = Tb @ (Cp[s] + Vb.T @ Ci)
                Cp[s] -= W; Q[piv][j] = Cp; Q[i][j] = Ci - Vb @ W
Qf = np.block([[Q[i][j] for j in range(q)] for i in range(p)])
o = float(np.linalg.norm(Qf.T@Qf - np.eye(n, dtype=FORM)))
print(f"n={n} {mode} orth={o:.3e}")
