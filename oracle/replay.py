"""Numeric oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module; the product path (paper_1303_3182_b200) never
does and has no CPU fallback.

The reference (pkg/src/tiledag) executes no numeric kernels
(pkg/README.md:11-12): its tiled builder only records which tile kernel runs
on which tiles, in which order (QrBuild, qr.py:376-532; kernel read/write
sets qr.py:421-481).  This module restates the numerics those kernels stand
for with LAPACK's tile kernels — the thesis' Table 3.1 / Alg. 3.2-3.3
 — replaying the reference trace in order:

  GEQRT(i,k)        a, T_G = dgeqrt(ib, A[i,k])
  UNMQR(i,k,j)      A[i,j] = dgemqrt(V_G(i,k), T_G(i,k), A[i,j], 'T')
  TTQRT(i,piv,k)    R_piv, V_E, T_E = dtpqrt(l=nb, ib, triu R_piv, triu R_i)
  TSQRT(i,piv,k)    R_piv, V_E, T_E = dtpqrt(l=0,  ib, triu R_piv, A[i,k])
  TTMQR/TSMQR       A[piv,j], A[i,j] = dtpmqrt(l, V_E, T_E, A[piv,j], A[i,j], 'T')

LAPACK comes from scipy 1.18.1 (scipy-openblas 0.3.30).  The result is
stored in exactly the device layout (tile-major, column-major tiles, R and
V_G sharing a tile, V_E over the eliminated tile, T as ib x nb per tile),
so device results can be compared element by element.  Parity is pinned
by (i) R uniqueness up to row signs against numpy.linalg.qr and (ii)
||A - QR|| and ||Q^T Q - I|| of the replay itself (tests/test_oracle.py).
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import lapack as L

GEQRT, TTQRT, TSQRT, UNMQR, TTMQR, TSMQR = range(6)  # include/tqr.h enum tqr_kind


class Replay:
    """Tile store + T factors in the device layout (0-based internally)."""

    def __init__(self, A, p, q, nb, ib=32):
        m, n = A.shape
        assert m == p * nb and n == q * nb, (A.shape, p, q, nb)
        self.p, self.q, self.nb, self.ib = p, q, nb, ib
        # tiles[i][j] Fortran-ordered nb x nb
        self.t = [[np.asfortranarray(A[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb]) for j in range(q)]
                  for i in range(p)]
        self.tg = {}
        self.te = {}

    # -- kernels -------------------------------------------------------------
    def geqrt(self, i, k):
        a, t, info = L.dgeqrt(self.ib, self.t[i][k])
        assert info == 0
        self.t[i][k] = np.asfortranarray(a)
        self.tg[(i, k)] = t

    def unmqr(self, i, k, j):
        c, info = L.dgemqrt(self.t[i][k], self.tg[(i, k)], self.t[i][j], side="L", trans="T")
        assert info == 0
        self.t[i][j] = np.asfortranarray(c)

    def _tpqrt(self, i, piv, k, l):
        rp = self.t[piv][k]
        ri = self.t[i][k]
        b_in = np.triu(ri) if l else ri
        a, b, t, info = L.dtpqrt(l, self.ib, np.triu(rp), b_in)
        assert info == 0
        # R_piv: upper triangle only (strict lower keeps V_G(piv,k))
        iu = np.triu_indices(self.nb)
        new = rp.copy(order="F")
        new[iu] = a[iu]
        self.t[piv][k] = new
        if l:  # V_E upper-triangular over R_i's place; strict lower keeps V_G(i,k)
            newi = ri.copy(order="F")
            newi[iu] = b[iu]
            self.t[i][k] = newi
        else:
            self.t[i][k] = np.asfortranarray(b)
        self.te[(i, k)] = t

    def ttqrt(self, i, piv, k):
        self._tpqrt(i, piv, k, self.nb)

    def tsqrt(self, i, piv, k):
        self._tpqrt(i, piv, k, 0)

    def _tpmqrt(self, i, piv, k, j, l, trans="T", store=None):
        st = self.t if store is None else store
        v = np.triu(self.t[i][k]) if l else self.t[i][k]
        a, b, info = L.dtpmqrt(l, v, self.te[(i, k)], st[piv][j], st[i][j], side="L", trans=trans)
        assert info == 0
        st[piv][j] = np.asfortranarray(a)
        st[i][j] = np.asfortranarray(b)

    def ttmqr(self, i, piv, k, j):
        self._tpmqrt(i, piv, k, j, self.nb)

    def tsmqr(self, i, piv, k, j):
        self._tpmqrt(i, piv, k, j, 0)

    # -- trace replay ----------------------------------------------------------
    def run(self, kinds, idx, limit=None):
        """Replay trace arrays (kind int, 1-based indices) in order."""
        n = len(kinds) if limit is None else min(limit, len(kinds))
        for t in range(n):
            kd = int(kinds[t])
            a, b, c, d = (int(x) - 1 for x in idx[t])
            if kd == GEQRT:
                self.geqrt(a, b)
            elif kd == UNMQR:
                self.unmqr(a, b, c)
            elif kd == TTQRT:
                self.ttqrt(a, b, c)
            elif kd == TSQRT:
                self.tsqrt(a, b, c)
            elif kd == TTMQR:
                self.ttmqr(a, b, c, d)
            else:
                self.tsmqr(a, b, c, d)
        return self

    # -- results ---------------------------------------------------------------
    def tiles_array(self):
        """(p*q*nb*nb,) in the device tile-major layout."""
        out = np.empty((self.q, self.p, self.nb * self.nb))
        for j in range(self.q):
            for i in range(self.p):
                out[j, i] = self.t[i][j].reshape(-1, order="F")
        return out.reshape(-1)

    def t_array(self, which):
        d = self.tg if which == "G" else self.te
        out = np.zeros((self.q, self.p, self.ib * self.nb))
        for (i, k), t in d.items():
            out[k, i] = np.asarray(t).reshape(-1, order="F")
        return out.reshape(-1)

    def r(self):
        n = self.q * self.nb
        R = np.zeros((n, n))
        for i in range(self.q):
            for j in range(i, self.q):
                R[i * self.nb:(i + 1) * self.nb, j * self.nb:(j + 1) * self.nb] = self.t[i][j]
        return np.triu(R)

    def form_q(self, kinds, idx):
        """Explicit Q (m x n): reflectors replayed in reverse with trans='N'
        on [I; 0] (dgemqrt / dtpmqrt semantics)."""
        p, q, nb = self.p, self.q, self.nb
        Q = [[np.zeros((nb, nb), order="F") for _ in range(q)] for _ in range(p)]
        for d in range(q):
            Q[d][d] = np.asfortranarray(np.eye(nb))
        for t in range(len(kinds) - 1, -1, -1):
            kd = int(kinds[t])
            a, b, c, _ = (int(x) - 1 for x in idx[t])
            if kd == GEQRT:
                for j in range(q):
                    cc, info = L.dgemqrt(self.t[a][b], self.tg[(a, b)], Q[a][j], side="L", trans="N")
                    Q[a][j] = np.asfortranarray(cc)
            elif kd in (TTQRT, TSQRT):
                l = nb if kd == TTQRT else 0
                for j in range(q):
                    self._tpmqrt(a, b, c, j, l, trans="N", store=Q)
        return np.block([[Q[i][j] for j in range(q)] for i in range(p)])


def replay_build(A, build, nb, ib=32, limit=None):
    """Replay a paper_1303_3182_b200 / tiledag-shaped QrBuild's trace."""
    kinds, idx, _ = build.trace_arrays()
    rp = Replay(A, build.p, build.q, nb, ib)
    rp.run(kinds, idx, limit)
    return rp


def row_sign_normalize(R):
    s = np.sign(np.diag(R))
    s[s == 0] = 1.0
    return R * s[:, None]
