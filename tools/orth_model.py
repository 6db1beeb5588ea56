"""Per-block-reflector orthogonality defect model (CPU, numpy).

Q_b = I - V T V^T is orthogonal iff T + T^T = T^T G T (G = V^T V).  For the
stored fp64 (V, T) of a panel block, ||Q_b^T Q_b - I||_F = sqrt(tr(C G C G))
with C = T + T^T - T^T G T, evaluated in long double.  Summed in quadrature
over every block reflector of a factorization, this models ||Q^T Q - I||_F
of the implicit Q (before Q formation).  Methods for tau / G / T:
  lapack : dlarfg tau, G and T in fp64 (sequential dots)
  dd_all : tau = 2/G_jj, G in double-double, T by dd back substitution
  dd_g   : tau = 2/G_jj, G in double-double rounded to fp64, T in fp64
  dd_diag: tau = 2/G_jj (dd), off-diagonal G and T in fp64
"""
import sys
import numpy as np

LD = np.longdouble


def householder_panel(A, tt_rows=None):
    """Unblocked Householder QR of A (rows x ib) in fp64, dlarfg-style.
    Returns V (unit diagonal implied, stored explicitly), tau."""
    A = A.copy()
    m, n = A.shape
    V = np.zeros_like(A)
    tau = np.zeros(n)
    for j in range(n):
        alpha = A[j, j]
        x = A[j + 1:, j]
        xn2 = float(np.dot(x, x))
        if xn2 == 0.0:
            V[j, j] = 1.0
            continue
        beta = -np.copysign(np.sqrt(alpha * alpha + xn2), alpha)
        t = (beta - alpha) / beta
        v = x / (alpha - beta)
        V[j, j] = 1.0
        V[j + 1:, j] = v
        tau[j] = t
        A[j, j] = beta
        A[j + 1:, j] = 0
        w = A[j, j + 1:] + v @ A[j + 1:, j + 1:]
        A[j, j + 1:] -= t * w
        A[j + 1:, j + 1:] -= t * np.outer(v, w)
    return V, tau


def t_fp64(V, tau, G=None):
    n = V.shape[1]
    if G is None:
        G = V.T @ V
    T = np.zeros((n, n))
    for j in range(n):
        T[j, j] = tau[j]
        for i in range(j - 1, -1, -1):
            s = 0.0
            for l in range(i + 1, j + 1):
                s += G[i, l] * T[l, j]
            T[i, j] = -tau[i] * s
    return T


def t_ld(V, G_ld):
    n = V.shape[1]
    T = np.zeros((n, n), dtype=LD)
    for j in range(n):
        T[j, j] = LD(2) / G_ld[j, j]
        for i in range(j - 1, -1, -1):
            s = LD(0)
            for l in range(i + 1, j + 1):
                s += G_ld[i, l] * T[l, j]
            T[i, j] = -T[i, i] * s
    return T


def defect(V, T):
    Vl = V.astype(LD)
    Tl = T.astype(LD)
    G = Vl.T @ Vl
    C = Tl + Tl.T - Tl.T @ G @ Tl
    M = C @ G
    return float(np.sqrt(abs(np.trace(M @ M))))


def block_defects(V, tau):
    Vl = V.astype(LD)
    Gl = Vl.T @ Vl
    out = {}
    out["lapack"] = defect(V, t_fp64(V, tau))
    Tdd = t_ld(V, Gl).astype(np.float64)
    out["dd_all"] = defect(V, Tdd)
    G64 = Gl.astype(np.float64)
    tau2 = (LD(2) / np.diagonal(Gl)).astype(np.float64)
    out["dd_g"] = defect(V, t_fp64(V, tau2, G64))
    out["dd_diag"] = defect(V, t_fp64(V, tau2, np.triu(V.T @ V, 1) + np.diag(np.diagonal(G64))))
    return out


def main():
    rng = np.random.default_rng(0)
    nb, ib = 256, 32
    res = {}
    for kind in ("GE", "TT"):
        acc = {}
        for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
            if kind == "GE":
                A = rng.standard_normal((nb, nb))
                for b in range(nb // ib):
                    r0 = b * ib
                    V, tau = householder_panel(A[r0:, r0:r0 + ib])
                    for k, v in block_defects(V, tau).items():
                        acc.setdefault(k, []).append(v)
            else:
                # TT block b: pivot rows r0..r0+ib of the upper triangle + bottom
                # triangle rows 0..r0+ib (dense upper-trapezoidal stacking)
                Rb = np.triu(rng.standard_normal((nb, nb)))
                for b in range(nb // ib):
                    r0 = b * ib
                    top = np.triu(rng.standard_normal((ib, ib)))
                    bot = Rb[:r0 + ib, r0:r0 + ib]
                    V, tau = householder_panel(np.vstack([top, bot]))
                    V[:ib] = np.eye(ib)  # the pivot part of a TT reflector is e_j
                    for k, v in block_defects(V, tau).items():
                        acc.setdefault(k, []).append(v)
        res[kind] = {k: float(np.sqrt(np.mean(np.square(v)))) for k, v in acc.items()}
    nge, ntt = 2080 * 8, 2016 * 8  # C3 block reflectors
    print("rms per-block defect:", res)
    for k in res["GE"]:
        tot = np.sqrt(nge * res["GE"][k] ** 2 + ntt * res["TT"][k] ** 2)
        print(f"{k:8s} modeled C3 ||Q^TQ-I||_F (implicit Q) = {tot:.3e}")


if __name__ == "__main__":
    main()
