"""Drop-in boundary: the reference's own objects (tiledag.EliminationList,
ElimEntry, WeightModel, Task traces) go through every entry point of this
package and give bit-identical results (qr.py:41-141, :535-545, :622-649;
taskgraph.py:78-146, :262-322).  CPU only: schedules, no kernels."""
import random

import pytest

import paper_1303_3182_b200 as P
from conftest import reference_tiledag

T = reference_tiledag()
pytestmark = pytest.mark.skipif(T is None, reason="reference tiledag package not available")


def _same_build(a, b):
    assert a.cp == b.cp and a.total_weight == b.total_weight and a.zeroed == b.zeroed
    assert dict(a.counts) == {k: v for k, v in b.counts.items()}
    assert [(t.kind, tuple(t.indices)) for t in a.trace] == [(t.kind, tuple(t.indices)) for t in b.trace]


TREES = [("greedy", 8, 4), ("fibonacci", 8, 4), ("sameh-kuck", 9, 5), ("greedy", 13, 13), ("fibonacci", 20, 7)]


@pytest.mark.parametrize("algo,p,q", TREES)
@pytest.mark.parametrize("family", ["TT", "TS"])
def test_tiled_build_accepts_reference_list(algo, p, q, family):
    ref_list = T.coarse_schedule(p, q, algo)[1]
    ours = P.tiled_build(ref_list, family)
    assert ours.elim is ref_list  # the caller's object is kept, as qr.py:521 does
    _same_build(ours, T.tiled_build(ref_list, family))
    _same_build(ours, P.tiled_build(P.coarse_schedule(p, q, algo)[1], family))
    assert [(t.kind, tuple(t.indices)) for t in P.tiled_graph(ref_list, family)] == \
        [(t.kind, tuple(t.indices)) for t in T.tiled_graph(ref_list, family)]


def test_reference_lists_with_reverse_entries():
    """User lists with reverse eliminations (i < piv), normalized / with_steps
    on the reference side, fed as reference objects."""
    rnd = random.Random(7)
    for trial in range(20):
        p, q = rnd.randint(2, 9), rnd.randint(1, 5)
        q = min(p, q)
        entries = []
        for k in range(1, q + 1):
            live = list(range(k, p + 1))
            while len(live) > 1:
                a, b = rnd.sample(live, 2)
                entries.append(T.ElimEntry(a, b, k))
                live.remove(a)
        lst = T.EliminationList(p, q, entries)
        try:
            lst.validate()
        except ValueError:
            with pytest.raises(ValueError):
                P.tiled_build(lst)
            continue
        lst = lst.with_steps()
        _same_build(P.tiled_build(lst, "TT"), T.tiled_build(lst, "TT"))


def test_invalid_reference_list_same_message():
    lst = T.EliminationList(4, 2, [T.ElimEntry(2, 1, 1), T.ElimEntry(2, 3, 1)])
    with pytest.raises(ValueError) as ref:
        T.tiled_build(lst)
    with pytest.raises(ValueError) as ours:
        P.tiled_build(lst)
    assert str(ours.value) == str(ref.value)


@pytest.mark.parametrize("algo", ["greedy", "asap", "grasap", "plasmatree", "fibonacci"])
def test_reference_weight_models(algo):
    bs = 3 if algo == "plasmatree" else None
    for wm in (T.WeightModel.qr_tt(), T.WeightModel.custom({T.GEQRT: 3, T.TTQRT: 1, T.UNMQR: 5, T.TTMQR: 4,
                                                             T.TSQRT: 7, T.TSMQR: 9})):
        ours = P.build_tree(10, 4, algo, bs=bs, weights=wm)
        ref = T.build_tree(10, 4, algo, bs=bs, weights=wm)
        _same_build(ours, ref)
    with pytest.raises(KeyError):
        P.build_tree(6, 3, "greedy", weights=T.WeightModel.custom({T.GEQRT: 1}))


@pytest.mark.parametrize("algo,family,p,q", [("greedy", "TT", 8, 4), ("sameh-kuck", "TS", 7, 3),
                                             ("grasap", "TT", 9, 4)])
def test_reference_trace_hazards_and_cp(algo, family, p, q):
    """build_from_trace / annotate_cp / asap_times on the reference's own Task
    trace and WeightModel (the C++ hazard rule)."""
    ref = T.build_tree(p, q, algo, family=family)
    g_ref = T.build_from_trace(ref.trace)
    g = P.build_from_trace(ref.trace)
    assert g.edges == g_ref.edges
    a = P.annotate_cp(g, ref.weights)
    b = T.annotate_cp(g_ref, ref.weights)
    assert a.cp_length == b.cp_length == ref.cp
    assert a.priority == b.priority and a.earliest == b.earliest
    fins, cp = P.asap_times(ref.trace, ref.weights)
    assert cp == ref.cp


def test_qrbuild_run_list_reference_list():
    ref_list = T.coarse_schedule(12, 6, "greedy")[1]
    b = P.QrBuild(12, 6, "TT", T.WeightModel.qr_tt()).run_list(ref_list)
    _same_build(b, T.QrBuild(12, 6, "TT").run_list(ref_list))
