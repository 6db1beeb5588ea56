"""Debug aid: tiny sub-diagonal input vs the LAPACK replay, per task prefix."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1303_3182_b200 as P
from paper_1303_3182_b200.engine import Plan
from oracle.replay import replay_build

for (p, q, nb, fam) in [(1, 1, 64, "TT"), (2, 1, 64, "TT"), (2, 2, 64, "TT"), (3, 2, 64, "TT"), (6, 3, 64, "TT")]:
    A0 = np.random.default_rng(31).standard_normal((p * nb, q * nb))
    A = np.triu(A0) + np.tril(A0, -1) * 1e-170
    b = P.build_tree(p, q, "greedy", family=fam)
    plan = Plan(b, nb)
    tiles, tg, te = plan.alloc()
    plan.pack(torch.from_numpy(A).cuda(), tiles)
    plan.factor(tiles, tg, te)
    torch.cuda.synchronize()
    t = tiles.cpu().numpy().reshape(q, p, nb, nb)
    rp = replay_build(A, b, nb)
    ref = rp.tiles_array().reshape(q, p, nb, nb)
    print(p, q, nb, [(i, j, float(np.abs(t[j, i] - ref[j, i]).max())) for j in range(q) for i in range(p)], flush=True)
    tgd = np.abs(tg.cpu().numpy() - rp.t_array("G")).max(); ted = np.abs(te.cpu().numpy() - rp.t_array("E")).max()
    print("   T diffs", tgd, ted)
    kinds, idx, _ = b.trace_arrays()
    print("   trace", [(int(k), tuple(int(x) for x in i[:3])) for k, i in zip(kinds, idx)][:12])
