"""Locate non-finite output of scaled inputs (debug aid for the panels'
scaled dnrm2-style path): factor small cases, report bad tiles."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1303_3182_b200 as P
from paper_1303_3182_b200.engine import Plan, TiledQR
from oracle.replay import replay_build

for (p, q, nb, algo) in [(1, 1, 64, "greedy"), (2, 1, 64, "greedy"), (1, 1, 256, "greedy"), (2, 1, 256, "greedy"),
                         (2, 2, 64, "greedy"), (6, 3, 64, "greedy")]:
    A = np.random.default_rng(31).standard_normal((p * nb, q * nb)) * 2.0 ** 664
    b = P.build_tree(p, q, algo)
    plan = Plan(b, nb)
    At = torch.from_numpy(A).cuda()
    tiles, tg, te = plan.alloc()
    plan.pack(At, tiles)
    plan.factor(tiles, tg, te)
    torch.cuda.synchronize()
    t = tiles.cpu().numpy().reshape(q, p, nb, nb)
    bad = [(i, j, int((~np.isfinite(t[j, i])).sum())) for j in range(q) for i in range(p) if not np.isfinite(t[j, i]).all()]
    tgb = int((~np.isfinite(tg.cpu().numpy())).sum()); teb = int((~np.isfinite(te.cpu().numpy())).sum())
    rp = replay_build(A, b, nb)
    ref = rp.tiles_array().reshape(q, p, nb, nb)
    err = np.nanmax(np.abs(np.where(np.isfinite(t), t, 0) - ref) / 2.0 ** 664)
    print(p, q, nb, "bad tiles", bad, "bad T", tgb, teb, "max scaled err", err, flush=True)
    if bad:
        i, j, _ = bad[0]
        nz = np.argwhere(~np.isfinite(t[j, i]))
        print("   first bad (col,row) in tile", (i, j), nz[:5].tolist())
