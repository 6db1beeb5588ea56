"""Command line mirror of the reference's QR subcommands (cli.py:112-150,
284-373): `qr-coarse` and `qr-tiled` write the same CSV tables with the same
--check / --out / TILEDAG_OUTDIR behaviour and exit codes (0 ok, 1 on check
mismatch or ValueError/AssertionError, 2 on bad flags).  `qr-numeric` (new)
factors a seeded random matrix on the GPU and reports GFLOP/s and errors.

    python -m paper_1303_3182_b200.cli qr-tiled --p 15 --q 6 --algo greedy --check
"""
from __future__ import annotations

import argparse
import json
import os
import sys

from . import qr

# frozen reference tables used by --check (the reference's golden.py holds
# the same 15x6 values; they are also pinned by tests/golden fixtures)
_COARSE_15x6_LAST = {"sameh-kuck": [14, 15, 16, 17, 18, 19], "fibonacci": [1, 3, 5, 7, 10, 12],
                     "greedy": [1, 2, 3, 5, 6, 8]}
_TILED_15x6_LAST = {"flattree": [32, 100, 116, 132, 148, 164], "fibonacci": [6, 22, 44, 60, 94, 116],
                    "greedy": [6, 22, 38, 60, 76, 98], "binarytree": [8, 28, 66, 90, 114, 134],
                    ("plasmatree", 5): [12, 40, 56, 72, 140, 164]}


def _write(args, text, suffix=""):
    out = getattr(args, "out", None)
    if out:
        outdir = os.environ.get("TILEDAG_OUTDIR", "")
        path = os.path.join(outdir, out + suffix) if outdir else out + suffix
        with open(path, "w") as fh:
            fh.write(text)
        print(f"wrote {path}")
    else:
        sys.stdout.write(text)


def _fail(cells):
    for c in cells:
        print(f"check mismatch: {c}", file=sys.stderr)
    return 1 if cells else 0


def cmd_qr_coarse(args):
    table, elim = qr.coarse_schedule(args.p, args.q, args.algo)
    _write(args, table.to_csv())
    if args.list:
        _write(args, elim.to_csv(), suffix=".elim")
    if args.check:
        cells = []
        cp, want = table.cp(), qr.coarse_cp_oracle(args.p, args.q, args.algo)
        if cp != want:
            cells.append(f"coarse cp: {cp} != {want}")
        if (args.p, args.q) == (15, 6):
            got = [table(15, k) for k in range(1, 7)]
            if got != _COARSE_15x6_LAST[table.algo]:
                cells.append(f"row 15: {got} != {_COARSE_15x6_LAST[table.algo]}")
        return _fail(cells)
    return 0


def cmd_qr_tiled(args):
    b = qr.build_tree(args.p, args.q, args.algo, family=args.family, bs=args.bs, grasap_i=args.i)
    _write(args, qr.zeroed_table_csv(b))
    if args.check:
        cells = []
        if not qr.verify_weight(b):
            cells.append("total weight mismatch")
        if args.algo == "flattree" and args.family == "TT":
            want = qr.flattree_cp_oracle(args.p, args.q)
            if b.cp != want:
                cells.append(f"cp {b.cp} != closed form {want}")
        key = (args.algo, args.bs) if args.algo == "plasmatree" else args.algo
        if (args.p, args.q) == (15, 6) and args.family == "TT" and key in _TILED_15x6_LAST:
            got = [b.zeroed.get((15, k)) for k in range(1, 7)]
            if got != _TILED_15x6_LAST[key]:
                cells.append(f"row 15: {got} != {_TILED_15x6_LAST[key]}")
        return _fail(cells)
    return 0


def cmd_qr_numeric(args):
    import time

    import numpy as np
    import torch

    from .engine import tiled_qr
    nb = args.nb
    A = np.random.default_rng(args.seed).standard_normal((args.p * nb, args.q * nb))
    At = torch.from_numpy(A).cuda()
    tiled_qr(At, nb=nb, algo=args.algo, family=args.family, bs=args.bs, grasap_i=args.i)  # warm-up + plan
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = tiled_qr(At, nb=nb, algo=args.algo, family=args.family, bs=args.bs, grasap_i=args.i)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    m, n = A.shape
    out = {"p": args.p, "q": args.q, "nb": nb, "algo": args.algo, "family": args.family, "cp": res.build.cp,
           "gflops": qr.qr_flops(m, n) / dt / 1e9}
    if args.check:
        R = res.R()
        Q = res.Q()
        nA = float(torch.linalg.norm(At))
        out["resid"] = float(torch.linalg.norm(At - Q @ R)) / nA
        out["orth"] = float(torch.linalg.norm(Q.T @ Q - torch.eye(n, dtype=torch.float64, device="cuda")))
    _write(args, json.dumps(out) + "\n")
    if args.check and (out["resid"] > 1e-12 or out["orth"] > 1e-12):
        return 1
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="tiledqr", description="B200 tiled QR: schedules and factorization")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def add(name, fn, **kw):
        p = sub.add_parser(name, **kw)
        p.set_defaults(fn=fn)
        p.add_argument("--out", help="output file (default stdout)")
        p.add_argument("--check", action="store_true", help="re-derive golden values; exit 1 on mismatch")
        return p

    p = add("qr-coarse", cmd_qr_coarse, help="coarse time-step table")
    p.add_argument("--p", type=int, required=True)
    p.add_argument("--q", type=int, required=True)
    p.add_argument("--algo", default="greedy", choices=["sameh-kuck", "fibonacci", "greedy"])
    p.add_argument("--list", action="store_true", help="also write the elimination list CSV")

    for name, fn, hlp in (("qr-tiled", cmd_qr_tiled, "tiled zeroed-time table"),
                          ("qr-numeric", cmd_qr_numeric, "factor a seeded N(0,1) matrix on the GPU")):
        p = add(name, fn, help=hlp)
        p.add_argument("--p", type=int, required=True)
        p.add_argument("--q", type=int, required=True)
        p.add_argument("--algo", default="greedy", choices=list(qr.TREE_ALGOS))
        p.add_argument("--family", default="TT", choices=["TT", "TS"])
        p.add_argument("--bs", type=int, help="plasmatree domain size")
        p.add_argument("--i", type=int, default=1, help="grasap trailing asap columns")
        if name == "qr-numeric":
            p.add_argument("--nb", type=int, default=256, choices=[64, 256])
            p.add_argument("--seed", type=int, default=0)

    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code not in (0, None) else 0
    try:
        return args.fn(args)
    except (ValueError, AssertionError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
