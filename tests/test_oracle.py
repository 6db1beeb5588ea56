"""Pin the numeric oracle (oracle/replay.py): the LAPACK replay of the
reference trace reproduces numpy.linalg.qr's R up to row signs and is a
backward-stable factorization (||A-QR||, ||Q^T Q - I|| small)."""
import numpy as np
import pytest

import paper_1303_3182_b200 as P
from oracle.replay import replay_build, row_sign_normalize


@pytest.mark.parametrize("algo,family,bs", [("greedy", "TT", None), ("flattree", "TS", None),
                                            ("fibonacci", "TT", None), ("plasmatree", "TT", 4),
                                            ("grasap", "TT", None), ("greedy", "TS", None),
                                            ("asap", "TT", None), ("binarytree", "TS", None)])
def test_replay_matches_dgeqrf(algo, family, bs):
    A = np.random.default_rng(1).standard_normal((512, 256))
    b = P.build_tree(8, 4, algo, family=family, bs=bs)
    rp = replay_build(A, b, 64)
    R = row_sign_normalize(rp.r())
    Rref = row_sign_normalize(np.linalg.qr(A, mode="r"))
    nA = np.linalg.norm(A)
    assert np.linalg.norm(R - Rref) <= 1e-13 * nA
    kinds, idx, _ = b.trace_arrays()
    Q = rp.form_q(kinds, idx)
    assert np.linalg.norm(A - Q @ rp.r()) / nA <= 1e-14
    assert np.linalg.norm(Q.T @ Q - np.eye(256)) <= 1e-13


def test_replay_ill_conditioned_fibonacci():
    """C4-shaped (Fibonacci, U diag(sigma) V^T, sigma 1..1e-12), reduced size."""
    rng = np.random.default_rng(3)
    m, n, nb = 1024, 512, 64
    U = np.linalg.qr(rng.standard_normal((m, n)))[0]
    V = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = (U * np.geomspace(1, 1e-12, n)) @ V.T
    b = P.build_tree(m // nb, n // nb, "fibonacci")
    rp = replay_build(A, b, nb)
    kinds, idx, _ = b.trace_arrays()
    Q = rp.form_q(kinds, idx)
    nA = np.linalg.norm(A)
    assert np.linalg.norm(A - Q @ rp.r()) / nA <= 1e-13
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-12
