import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1303_3182_b200 as P
from paper_1303_3182_b200.engine import Plan
from oracle.replay import replay_build
for (p, q, nb, algo, fam) in [(2, 1, 64, "greedy", "TT"), (6, 3, 64, "greedy", "TT"), (6, 3, 64, "flattree", "TS")]:
    A0 = np.random.default_rng(31).standard_normal((p * nb, q * nb))
    m, n = A0.shape
    A = A0.copy(); A[:, :nb] = np.triu(A0[:, :nb]) + np.tril(A0[:, :nb], -1) * 1e-170
    b = P.build_tree(p, q, algo, family=fam)
    plan = Plan(b, nb)
    tiles, tg, te = plan.alloc()
    plan.pack(torch.from_numpy(A).cuda(), tiles)
    plan.factor(tiles, tg, te)
    torch.cuda.synchronize()
    t = tiles.cpu().numpy().reshape(q, p, nb, nb)
    rp = replay_build(A, b, nb)
    ref = rp.tiles_array().reshape(q, p, nb, nb)
    for j in range(q):
        for i in range(p):
            d = np.abs(t[j, i] - ref[j, i])
            if d.max() > 1e-12:
                c, r = np.unravel_index(np.argmax(d), d.shape)
                print(p, q, algo, "tile", (i + 1, j + 1), "max", d.max(), "at col,row", (int(c), int(r)), "ours", t[j, i][c, r], "ref", ref[j, i][c, r], flush=True)
    for nm, arr in (("G", tg), ("E", te)):
        d = np.abs(arr.cpu().numpy() - rp.t_array(nm))
        if d.max() > 1e-12:
            k = int(np.argmax(d)); print("  T", nm, "max", d.max(), "flat idx", k, "ours", arr.cpu().numpy()[k], "ref", rp.t_array(nm)[k])
    print(p, q, algo, "done", flush=True)
