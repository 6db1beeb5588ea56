"""Debug aid: run trace prefixes of the 2x2 tiny-below case, compare tiles
with the LAPACK replay after each prefix."""
import sys, os, ctypes as C
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1303_3182_b200 as P
from paper_1303_3182_b200 import _lib
from paper_1303_3182_b200.qr import QrBuild
from paper_1303_3182_b200.engine import Plan
from oracle.replay import Replay

p, q, nb = 2, 2, 64
A0 = np.random.default_rng(31).standard_normal((p * nb, q * nb))
A = np.triu(A0) + np.tril(A0, -1) * 1e-170
b = P.build_tree(p, q, "greedy")
kinds, idx, _ = b.trace_arrays()
for n in range(1, len(kinds) + 1):
    h = C.c_void_p()
    k = np.ascontiguousarray(kinds[:n]); ix = np.ascontiguousarray(idx[:n])
    _lib.check(_lib.lib().tqr_trace_build(p, q, k.ctypes.data_as(_lib.i8p), _lib.ptr_i32(ix), n, C.byref(h)))
    mb = QrBuild.__new__(QrBuild)
    mb.__dict__.update(p=p, q=q, family="TT", keep_trace=True, _h=h, record_updates=False)
    plan = Plan(mb, nb)
    tiles, tg, te = plan.alloc()
    plan.pack(torch.from_numpy(A).cuda(), tiles)
    plan.factor(tiles, tg, te)
    torch.cuda.synchronize()
    t = tiles.cpu().numpy().reshape(q, p, nb, nb)
    rp = Replay(A, p, q, nb).run(k, ix)
    ref = rp.tiles_array().reshape(q, p, nb, nb)
    d = [(i, j, float(np.abs(t[j, i] - ref[j, i]).max())) for j in range(q) for i in range(p)]
    print(n, int(kinds[n - 1]), tuple(int(x) for x in idx[n - 1]), d, flush=True)
    if n == len(kinds):
        tt = t[1, 1].T; rr = ref[1, 1].T  # row-major views [row][col]
        for c in range(nb):
            e = np.abs(tt[:, c] - rr[:, c]).max()
            if e > 1e-12:
                print("first bad column", c, "err", e, "ours diag", tt[c, c], "ref diag", rr[c, c],
                      "x max", np.abs(rr[c + 1:, c]).max() if c + 1 < nb else 0)
                break
