"""How much of ||Q^T Q - I||_F at n = 16384 is the check's own rounding?
The Gram Q^T Q is formed twice: one DGEMM over all m rows (the usual check),
and as a Kahan-compensated sum of DGEMMs over row blocks of BLK rows (each
block's partial sums stay small, the cross-block sum is compensated).  Both
for our Q (tiled_qr, C3 Greedy/TT, seed 2) and for cuSOLVER's
(torch.linalg.qr).  Test infrastructure only; prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_3182_b200.engine import tiled_qr  # noqa: E402

BLK = int(os.environ.get("BLK", "128"))


def orth_plain(Q):
    G = Q.T @ Q
    G.diagonal().sub_(1.0)
    return torch.linalg.norm(G).item()


def orth_compensated(Q, blk=BLK):
    n = Q.shape[1]
    S = torch.zeros((n, n), dtype=torch.float64, device=Q.device)
    c = torch.zeros_like(S)
    for r0 in range(0, Q.shape[0], blk):
        q = Q[r0:r0 + blk]
        y = torch.mm(q.T, q)
        y.sub_(c)
        t = S + y
        c = (t - S).sub_(y)
        S = t
        del y, t
    S.diagonal().sub_(1.0)  # exact (Sterbenz) on the ~1 diagonal
    S.sub_(c)
    return torch.linalg.norm(S).item()


def main():
    out = {"blk": BLK}
    for n in [int(x) for x in os.environ.get("SIZES", "8192,16384").split(",")]:
        A = np.random.default_rng(2).standard_normal((n, n))
        At = torch.from_numpy(A).cuda()
        res = tiled_qr(At, nb=256, algo="greedy")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        Q = res.Q()
        e1.record()
        torch.cuda.synchronize()
        R = res.R()
        rec = {"ours": {"form_q_ms": e0.elapsed_time(e1), "orth_plain": orth_plain(Q), "orth_comp": orth_compensated(Q),
                        "resid": (torch.linalg.norm(At - Q @ R) / torch.linalg.norm(At)).item()}}
        del Q, R, res
        torch.cuda.empty_cache()
        if os.environ.get("SKIP_CUSOLVER"):
            out[n] = rec
            print(json.dumps({n: rec}), file=sys.stderr, flush=True)
            continue
        Qc, Rc = torch.linalg.qr(At)
        rec["cusolver"] = {"orth_plain": orth_plain(Qc), "orth_comp": orth_compensated(Qc),
                           "resid": (torch.linalg.norm(At - Qc @ Rc) / torch.linalg.norm(At)).item()}
        del Qc, Rc, At
        torch.cuda.empty_cache()
        out[n] = rec
        print(json.dumps({n: rec}), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
