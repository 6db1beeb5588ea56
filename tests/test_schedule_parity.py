"""Bit-exact schedule parity: the C++ compiler (via the reference-shaped
Python API) against golden vectors generated from the reference itself
(tests/golden/make_golden.py imports pkg/src/tiledag)."""
import pytest

import paper_1303_3182_b200 as P
from paper_1303_3182_b200 import WeightModel

from _digest import build_digest, elim_flat, elim_sha, zeroed_flat, zeroed_sha


def _check_record(b, rec, what):
    assert b.cp == rec["cp"], what
    assert b.total_weight == rec["total_weight"], what
    assert b.counts == rec["counts"], what
    if "ntasks" in rec:
        assert len(b.trace) == rec["ntasks"], what
        assert build_digest(b) == rec["trace_sha"], what
    if "elim" in rec:
        assert elim_flat(b.elim) == rec["elim"], what
    if "zeroed" in rec:
        assert zeroed_flat(b) == rec["zeroed"], what


def test_coarse_tables_and_lists(golden):
    for key, rec in golden["coarse"].items():
        algo, p, q = key.split("/")
        p, q = int(p), int(q)
        table, elim = P.coarse_schedule(p, q, algo)
        assert elim_flat(elim) == rec["elim"], key
        assert table.cp() == rec["cp"], key
        assert table.x == rec["x"], key
        assert [[i, k, s] for (i, k), s in sorted(table.steps.items())] == rec["steps"], key
        assert P.coarse_cp_oracle(p, q, algo) == rec["oracle_cp"], key
        elim.validate()
        table.validate(elim)


def test_build_tree_all_trees_families(golden):
    for key, rec in golden["trees"].items():
        algo, fam, bs, gi, p, q = key.split("/")
        bs = None if bs == "None" else int(bs)
        b = P.build_tree(int(p), int(q), algo, family=fam, bs=bs, grasap_i=int(gi))
        _check_record(b, rec, key)
        assert P.verify_weight(b), key


def test_custom_weight_models(golden):
    w = WeightModel.custom({"GEQRT": 3, "TTQRT": 1, "UNMQR": 5, "TTMQR": 4, "TSQRT": 7, "TSMQR": 9})
    for key, rec in golden["custom_weights"].items():
        algo, fam, p, q = key.split("/")
        b = P.build_tree(int(p), int(q), algo, family=fam, weights=w)
        _check_record(b, rec, key)


def test_user_lists_reverse_entries(golden):
    for n, rec in enumerate(golden["random_lists"]):
        p, q = rec["p"], rec["q"]
        f = rec["elim"]
        lst = P.EliminationList(p, q, [P.ElimEntry(*f[t:t + 4]) for t in range(0, len(f), 4)])
        lst.validate()
        assert elim_flat(lst.with_steps()) == rec["with_steps"], n
        assert elim_flat(lst.normalized()) == rec["normalized"], n
        for fam in ("TT", "TS"):
            b = P.tiled_build(lst, family=fam)
            _check_record(b, rec[fam], (n, fam))


def test_validate_messages(golden):
    for rec in golden["validate_errors"]:
        lst = P.EliminationList(rec["p"], rec["q"], [P.ElimEntry(i, v, k) for i, v, k in rec["elim"]])
        if rec["error"] is None:
            assert lst.validate()
        else:
            with pytest.raises(ValueError) as ei:
                lst.validate()
            assert str(ei.value) == rec["error"]


def test_hazard_dag(golden):
    for key, rec in golden["hazard"].items():
        algo, fam, p, q = key.split("/")
        b = P.build_tree(int(p), int(q), algo, family=fam)
        g = P.build_from_trace(b.trace)
        assert len(g.edges) == rec["nedges"], key
        if rec["edges"] is not None:
            assert [list(e) for e in g.edges] == rec["edges"], key
        ann = P.annotate_cp(g, b.weights)
        assert ann.cp_length == rec["cp"] == b.cp, key
        assert [ann.priority[t.id] for t in b.trace] == rec["priority"], key
        assert [ann.earliest[t.id] for t in b.trace] == rec["earliest"], key
        # builder times are the hazard-DAG earliest times (test_qr_tiled.py:277-296)
        _, _, fin = b.trace_arrays()
        assert [ann.earliest[t] + b.weights.of(b.trace[t]) for t in range(len(b.trace))] == fin.tolist()


def test_p40_columns(golden):
    g = golden["p40"]
    for q in range(1, 41):
        assert P.build_tree(40, q, "greedy", keep_trace=False).cp == g["greedy"][q - 1]
        assert P.build_tree(40, q, "fibonacci", keep_trace=False).cp == g["fibonacci"][q - 1]
        assert P.build_tree(40, q, "plasmatree", bs=10, keep_trace=False).cp == g["plasmatree_bs10"][q - 1]
        assert P.build_tree(40, q, "asap", keep_trace=False).cp == g["asap"][q - 1]
        assert P.build_tree(40, q, "grasap", keep_trace=False).cp == g["grasap"][q - 1]


@pytest.mark.parametrize("name", ["C1", "C2-flattree-TS", "C2-fibonacci", "C2-greedy", "C2-plasmatree4",
                                  "C2-grasap", "C3", "C4", "C5", "C5-local2", "C5-local4", "C5-local8"])
def test_baseline_configs(golden, name):
    rec = golden["configs"][name]
    b = P.build_tree(rec["p"], rec["q"], rec["algo"], family=rec["family"], bs=rec["bs"])
    _check_record(b, rec, name)
    assert elim_sha(b.elim) == rec["elim_sha"]
    assert zeroed_sha(b) == rec["zeroed_sha"]
    assert len(b.elim) == rec["nelim"]
    assert max(e.step for e in b.elim) == rec["nsteps"]


def test_error_paths():
    with pytest.raises(ValueError, match="need p >= q >= 1"):
        P.build_tree(3, 4, "greedy")
    with pytest.raises(ValueError, match="unknown algorithm 'nope'"):
        P.build_tree(4, 3, "NOPE")
    with pytest.raises(ValueError, match="plasmatree needs a domain size bs"):
        P.build_tree(4, 3, "plasmatree")
    with pytest.raises(ValueError, match="domain size must satisfy"):
        P.plasmatree_list(5, 3, 6)
    with pytest.raises(ValueError, match="Asap is defined over TT kernels"):
        P.build_tree(4, 3, "asap", family="TS")
    with pytest.raises(ValueError, match="GrASAP is defined over TT kernels"):
        P.build_tree(4, 3, "grasap", family="TS")
    with pytest.raises(ValueError, match="need 1 <= i <= q"):
        P.build_tree(4, 3, "grasap", grasap_i=5)
    with pytest.raises(ValueError, match="kernel family"):
        P.build_tree(4, 3, "greedy", family="XX")
    with pytest.raises(ValueError, match="unknown coarse algorithm"):
        P.coarse_schedule(4, 3, "binarytree")
    bad = P.EliminationList(3, 2, P.coarse_schedule(3, 2, "greedy")[1].entries[:2])
    with pytest.raises(ValueError, match="incomplete"):
        P.tiled_graph(bad, "TT")


def test_csv_round_trip():
    _, elim = P.coarse_schedule(6, 3, "greedy")
    text = elim.to_csv()
    assert text.splitlines()[0] == "k,i,piv,step"
    back = P.EliminationList.from_csv(6, 3, text)
    assert elim_flat(back) == elim_flat(elim)
