"""The CPU baseline's DAG-parallel LAPACK replay (oracle/cpu_baseline.py)
executes the reference trace exactly: same tiles as the sequential replay
(oracle/replay.py), for traces built by the reference itself."""
import numpy as np
import pytest
from threadpoolctl import threadpool_limits

from conftest import reference_tiledag
from oracle.cpu_baseline import DagReplay, edges_of, trace_arrays_of
from oracle.replay import Replay

T = reference_tiledag()


@pytest.mark.skipif(T is None, reason="reference tiledag package not available")
@pytest.mark.parametrize("algo,family,p,q,nb", [("greedy", "TT", 6, 4, 64), ("sameh-kuck", "TS", 5, 3, 64),
                                                ("fibonacci", "TT", 7, 7, 32)])
def test_dag_replay_matches_sequential(algo, family, p, q, nb):
    A = np.random.default_rng(3).standard_normal((p * nb, q * nb))
    b = T.build_tree(p, q, algo, family=family)
    kinds, idx = trace_arrays_of(b)
    dr = DagReplay(A, p, q, nb, kinds, idx, edges_of(b, T), workers=3)
    try:
        n = 0
        while not dr.finished():
            fl, dt, cnt = dr.run_for(0.01)
            n += cnt
        assert n == len(kinds)
        with threadpool_limits(1):
            rp = Replay(A, p, q, nb).run(kinds, idx)
        got = np.stack([dr.tiles[j * p + i].T for j in range(q) for i in range(p)])
        ref = np.stack([rp.t[i][j] for j in range(q) for i in range(p)])
        assert np.array_equal(got, ref)
    finally:
        dr.close()
