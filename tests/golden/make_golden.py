"""Generate the schedule golden fixtures from the reference itself.

Runs ONLY in the build container, where the read-only reference lives at
/root/reference (it does not exist on the GPU box).  It imports the
reference package `tiledag` (pkg/src/tiledag) and records, for many shapes,
trees, kernel families and weight models, the exact outputs of its public
API: elimination lists with coarse steps, zeroed-time tables, critical
paths, kernel counts and a digest of the full task trace.  The committed
fixtures (schedules.json.gz) are what tests/ compares the product (the C++
schedule compiler behind paper_1303_3182_b200) and oracle/schedule.py with.

Usage:  python tests/golden/make_golden.py
"""
import gzip
import hashlib
import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import tiledag as T  # noqa: E402
from tiledag import cli as T_cli  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "schedules.json.gz")


def trace_digest(trace):
    """sha256 over 'KIND:i,j,k;' for every task in trace order."""
    h = hashlib.sha256()
    for t in trace:
        h.update(f"{t.kind}:{','.join(str(x) for x in t.indices)};".encode())
    return h.hexdigest()


def edges_digest(graph):
    h = hashlib.sha256()
    for u, v, c in graph.edges:
        h.update(f"{u}>{v}:{c};".encode())
    return h.hexdigest(), len(graph.edges)


def elim_flat(elim):
    out = []
    for e in elim:
        out += [e.i, e.piv, e.k, e.step]
    return out


def zeroed_flat(b):
    return [[i, k, v] for (i, k), v in sorted(b.zeroed.items())]


def record(b, with_list=True, with_zeroed=True):
    r = {"cp": b.cp, "total_weight": b.total_weight,
         "counts": dict(b.counts)}
    if b.trace is not None:
        r["ntasks"] = len(b.trace)
        r["trace_sha"] = trace_digest(b.trace)
    if with_list:
        r["elim"] = elim_flat(b.elim)
    if with_zeroed:
        r["zeroed"] = zeroed_flat(b)
    return r


def custom_weights():
    return T.WeightModel.custom({"GEQRT": 3, "TTQRT": 1, "UNMQR": 5,
                                 "TTMQR": 4, "TSQRT": 7, "TSMQR": 9})


def random_list(p, q, rng, rev_cols):
    entries = []
    for k in range(1, min(p, q) + 1):
        rows = list(range(k, p + 1))
        while len(rows) > 1:
            a, b = sorted(rng.sample(range(len(rows)), 2))
            lo, hi = rows[a], rows[b]
            if k in rev_cols and lo > k and rng.random() < 0.5:
                entries.append(T.ElimEntry(lo, hi, k))
                rows.remove(lo)
            else:
                entries.append(T.ElimEntry(hi, lo, k))
                rows.remove(hi)
    return T.EliminationList(p, q, entries)


def main():
    g = {"generator": "tests/golden/make_golden.py", "reference": "tiledag (pkg/src)",
         "digest": "sha256 over 'KIND:idx,..;' per task in trace order"}

    # 1. coarse tables + lists (qr.py:279-297), 1<=q<=p<=16
    coarse = {}
    for p in range(1, 17):
        for q in range(1, p + 1):
            for algo in ("sameh-kuck", "fibonacci", "greedy"):
                table, elim = T.coarse_schedule(p, q, algo)
                coarse[f"{algo}/{p}/{q}"] = {
                    "elim": elim_flat(elim), "cp": table.cp(), "x": table.x,
                    "steps": [[i, k, s] for (i, k), s in sorted(table.steps.items())],
                    "oracle_cp": T.coarse_cp_oracle(p, q, algo)}
    g["coarse"] = coarse

    # 2. build_tree for every tree/family, 1<=q<=p<=12 (qr.py:622-649)
    trees = {}
    for p in range(1, 13):
        for q in range(1, p + 1):
            variants = [("flattree", "TT", None, 1), ("flattree", "TS", None, 1),
                        ("fibonacci", "TT", None, 1), ("fibonacci", "TS", None, 1),
                        ("greedy", "TT", None, 1), ("greedy", "TS", None, 1),
                        ("binarytree", "TT", None, 1), ("binarytree", "TS", None, 1),
                        ("asap", "TT", None, 1), ("grasap", "TT", None, 1)]
            for bs in sorted(b for b in {1, 2, 3, max(1, p // 2), p} if b <= p):
                variants.append(("plasmatree", "TT", bs, 1))
                variants.append(("plasmatree", "TS", bs, 1))
            for gi in range(2, q + 1):
                variants.append(("grasap", "TT", None, gi))
            for algo, fam, bs, gi in variants:
                b = T.build_tree(p, q, algo, family=fam, bs=bs, grasap_i=gi)
                trees[f"{algo}/{fam}/{bs}/{gi}/{p}/{q}"] = record(b)
    g["trees"] = trees

    # 3. custom weight model (weight-dependent Asap/GrASAP lists, qr.py:551-611)
    cw = {}
    for p, q in ((5, 3), (8, 4), (12, 5), (15, 6), (20, 6)):
        for algo, fam in (("asap", "TT"), ("grasap", "TT"), ("greedy", "TT"),
                          ("greedy", "TS"), ("flattree", "TS")):
            b = T.build_tree(p, q, algo, family=fam, weights=custom_weights())
            cw[f"{algo}/{fam}/{p}/{q}"] = record(b)
    g["custom_weights"] = cw

    # 4. user lists incl. reverse eliminations through tiled_build (qr.py:535-540),
    #    normalized() (qr.py:85-116), with_steps() (qr.py:118-127)
    rng = random.Random(2)
    rl = []
    for n in range(60):
        p = rng.randint(2, 9)
        q = rng.randint(1, p)
        rev = set(range(1, q + 1)) if n % 2 else {min(p, q)}
        lst = random_list(p, q, rng, rev)
        rec = {"p": p, "q": q, "elim": elim_flat(lst),
               "with_steps": elim_flat(lst.with_steps()),
               "normalized": elim_flat(lst.normalized())}
        for fam in ("TT", "TS"):
            b = T.tiled_build(lst, family=fam)
            rec[fam] = record(b, with_list=False)
        rl.append(rec)
    g["random_lists"] = rl

    # 5. validate() rejections and their messages (qr.py:56-83)
    bad_cases = [
        (3, 2, [(3, 2, 1), (3, 2, 2), (2, 1, 1)]),
        (3, 1, [(2, 1, 1), (3, 2, 1)]),
        (3, 1, [(2, 1, 1)]),
        (3, 2, [(2, 3, 2)]),
        (3, 1, [(2, 2, 1)]),
        (3, 2, [(2, 1, 1), (3, 1, 1), (3, 2, 2)]),
        (4, 2, [(2, 1, 1), (2, 1, 1)]),
        (4, 2, [(2, 1, 1), (3, 1, 1), (4, 1, 1), (3, 1, 2)]),
        (4, 4, [(5, 1, 1)]),
        (4, 2, [(2, 1, 0)]),
    ]
    bad = []
    for p, q, ents in bad_cases:
        lst = T.EliminationList(p, q, [T.ElimEntry(i, v, k) for i, v, k in ents])
        try:
            lst.validate()
            msg = None
        except ValueError as e:
            msg = str(e)
        bad.append({"p": p, "q": q, "elim": [list(e) for e in ents], "error": msg})
    g["validate_errors"] = bad

    # 6. hazard DAG (taskgraph.py:262-322) and Backflow (taskgraph.py:338-362)
    hz = {}
    for p, q, algo, fam in ((5, 3, "greedy", "TT"), (6, 4, "flattree", "TT"),
                            (7, 3, "asap", "TT"), (6, 3, "binarytree", "TT"),
                            (5, 5, "grasap", "TT"), (5, 3, "greedy", "TS"),
                            (8, 4, "fibonacci", "TS"), (8, 4, "greedy", "TT")):
        b = T.build_tree(p, q, algo, family=fam)
        gr = T.build_from_trace(b.trace)
        ann = T.annotate_cp(gr, b.weights)
        dig, ne = edges_digest(gr)
        hz[f"{algo}/{fam}/{p}/{q}"] = {
            "edges_sha": dig, "nedges": ne, "cp": ann.cp_length,
            "edges": [[u, v, c] for u, v, c in gr.edges] if len(gr.edges) < 400 else None,
            "priority": [ann.priority[t.id] for t in b.trace],
            "earliest": [ann.earliest[t.id] for t in b.trace]}
    g["hazard"] = hz

    # 7. p=40 critical-path columns (acceptance criterion 9 shape)
    g["p40"] = {
        "greedy": [T.build_tree(40, q, "greedy", keep_trace=False).cp for q in range(1, 41)],
        "fibonacci": [T.build_tree(40, q, "fibonacci", keep_trace=False).cp for q in range(1, 41)],
        "plasmatree_bs10": [T.build_tree(40, q, "plasmatree", bs=10, keep_trace=False).cp
                            for q in range(1, 41)],
        "asap": [T.build_tree(40, q, "asap", keep_trace=False).cp for q in range(1, 41)],
        "grasap": [T.build_tree(40, q, "grasap", keep_trace=False).cp for q in range(1, 41)],
    }

    # 8. BASELINE configs (C1..C5) summaries
    cfg = {}
    for name, p, q, algo, fam, bs in (
            ("C1", 8, 4, "greedy", "TT", None),
            ("C2-flattree-TS", 8, 4, "flattree", "TS", None),
            ("C2-fibonacci", 8, 4, "fibonacci", "TT", None),
            ("C2-greedy", 8, 4, "greedy", "TT", None),
            ("C2-plasmatree4", 8, 4, "plasmatree", "TT", 4),
            ("C2-grasap", 8, 4, "grasap", "TT", None),
            ("C3", 64, 64, "greedy", "TT", None),
            ("C4", 32, 16, "fibonacci", "TT", None),
            ("C5", 8192, 8, "greedy", "TT", None),
            ("C5-local2", 4096, 8, "greedy", "TT", None),
            ("C5-local4", 2048, 8, "greedy", "TT", None),
            ("C5-local8", 1024, 8, "greedy", "TT", None)):
        b = T.build_tree(p, q, algo, family=fam, bs=bs)
        r = record(b, with_list=(p * q <= 4096), with_zeroed=(p * q <= 4096))
        h = hashlib.sha256()
        for e in b.elim:
            h.update(f"{e.k},{e.i},{e.piv},{e.step};".encode())
        r["elim_sha"] = h.hexdigest()
        r["nelim"] = len(b.elim)
        r["nsteps"] = max((e.step for e in b.elim), default=0)
        zh = hashlib.sha256()
        for (i, k), v in sorted(b.zeroed.items()):
            zh.update(f"{i},{k},{v};".encode())
        r["zeroed_sha"] = zh.hexdigest()
        r.update({"p": p, "q": q, "algo": algo, "family": fam, "bs": bs})
        cfg[name] = r
    g["configs"] = cfg

    # 8b. tall-skinny composite lists (local Greedy per shard + binary TT
    #     merges) through the reference's validate() and
    #     tiled_build(): validity, CP, total weight, trace digest
    def merge_pairs(q, row_a, rows_b):
        # restated from dist.merge_pairs: per column the two earliest-ready
        # live rows pair (R_a's row survives, else the lower row); costs
        # TTQRT 15, TTMQR 2, GEQRT 15; emitted in simulated start order
        import heapq
        ev, carry = [], []
        for k in range(1, q + 1):
            live = [(0, k), (0, q + k)] + carry
            carry = []
            heapq.heapify(live)
            while len(live) > 1:
                t1, r1 = heapq.heappop(live)
                t2, r2 = heapq.heappop(live)
                s = max(t1, t2)
                piv, tgt = (r1, r2) if (r1 == k or (r2 != k and r1 < r2)) else (r2, r1)
                ev.append((s, tgt, piv, k))
                heapq.heappush(live, (s + 15, piv))
                carry.append((s + 32, tgt))
        ev.sort()
        row = lambda r: row_a(r) if r <= q else rows_b(r - q)  # noqa: E731
        return [T.ElimEntry(row(t), row(v), k) for _, t, v, k in ev]

    comp = {}
    for p, q, G in ((64, 8, 8), (16, 4, 2), (16, 4, 4), (8192, 8, 1), (8192, 8, 2), (8192, 8, 8)):
        P = p // G
        _, local = T.coarse_schedule(P, q, "greedy")
        ents = []
        for s in range(G):
            ents += [T.ElimEntry(e.i + s * P, e.piv + s * P, e.k) for e in local]
        stride = 1
        while stride < G:
            for a in range(0, G, 2 * stride):
                b = a + stride
                if b < G:
                    ents += merge_pairs(q, lambda k, a=a: a * P + k, lambda i, b=b: b * P + i)
            stride *= 2
        lst = T.EliminationList(p, q, ents).with_steps()
        lst.validate()
        b = T.tiled_build(lst, keep_trace=(p <= 64))
        h = hashlib.sha256()
        for e in lst:
            h.update(f"{e.k},{e.i},{e.piv},{e.step};".encode())
        rec = {"cp": b.cp, "total_weight": b.total_weight, "elim_sha": h.hexdigest(), "nelim": len(lst)}
        if b.trace is not None:
            rec["trace_sha"] = trace_digest(b.trace)
        comp[f"{p}/{q}/{G}"] = rec
    g["composite"] = comp

    # 9. CLI outputs (cli.py:112-150)
    import contextlib
    import io
    clio = {}
    for argv in (["qr-coarse", "--p", "15", "--q", "6", "--algo", "greedy", "--check"],
                 ["qr-coarse", "--p", "9", "--q", "4", "--algo", "fibonacci"],
                 ["qr-tiled", "--p", "15", "--q", "6", "--algo", "greedy", "--check"],
                 ["qr-tiled", "--p", "15", "--q", "6", "--algo", "plasmatree", "--bs", "5"],
                 ["qr-tiled", "--p", "10", "--q", "4", "--algo", "grasap"],
                 ["qr-tiled", "--p", "8", "--q", "4", "--algo", "flattree", "--family", "TS"],
                 ["qr-coarse", "--p", "3", "--q", "5"]):
        buf, ebuf = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(ebuf):
            rc = T_cli.main(argv)
        clio[" ".join(argv)] = {"rc": rc, "out": buf.getvalue(), "err": ebuf.getvalue()}
    g["cli"] = clio

    with gzip.open(OUT, "wt") as fh:
        json.dump(g, fh, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
