"""Determinism soak: repeat factorizations and compare every tile and T factor
bit for bit with the first run (a shared-memory or flag race in the kernels
would show up as run-to-run differences)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1303_3182_b200 as P  # noqa: E402
from paper_1303_3182_b200.engine import Plan  # noqa: E402

CASES = [  # (p, q, nb, algo, family, reps)
    (32, 16, 256, "fibonacci", "TT", 40),
    (64, 64, 256, "greedy", "TT", 8),
    (24, 8, 256, "flattree", "TS", 30),
    (40, 12, 128, "greedy", "TT", 30),
    (48, 16, 64, "binarytree", "TT", 30),
    (1024, 8, 256, "greedy", "TT", 6),
]
bad = 0
for p, q, nb, algo, fam, reps in CASES:
    A = torch.from_numpy(np.random.default_rng(p * q).standard_normal((p * nb, q * nb))).cuda()
    plan = Plan(P.build_tree(p, q, algo, family=fam), nb)
    tiles, tg, te = plan.alloc()
    ref = None
    for r in range(reps):
        plan.pack(A, tiles)
        plan.factor(tiles, tg, te)
        torch.cuda.synchronize()
        cur = (tiles.clone(), tg.clone(), te.clone())
        if ref is None:
            ref = cur
        elif not all(torch.equal(a, b) for a, b in zip(ref, cur)):
            bad += 1
            print(f"MISMATCH {p}x{q} nb={nb} {algo}/{fam} run {r}", flush=True)
    print(f"{p}x{q} nb={nb} {algo}/{fam}: {reps} runs identical" if not bad else "...", flush=True)
print("soak", "FAILED" if bad else "ok")
sys.exit(1 if bad else 0)
