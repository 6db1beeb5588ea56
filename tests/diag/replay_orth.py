"""Orthogonality / residual of the LAPACK tile replay (oracle) of the C3
Greedy trace at reduced and full size, on the CPU (reference numbers)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1303_3182_b200 as P
from oracle.replay import replay_build

for n in [int(x) for x in os.environ.get("SIZES", "8192").split(",")]:
    t0 = time.time()
    A = np.random.default_rng(2).standard_normal((n, n))
    b = P.build_tree(n // 256, n // 256, "greedy")
    rp = replay_build(A, b, 256)
    kinds, idx, _ = b.trace_arrays()
    Q = rp.form_q(kinds, idx)
    R = rp.r()
    orth = np.linalg.norm(Q.T @ Q - np.eye(n))
    resid = np.linalg.norm(A - Q @ R) / np.linalg.norm(A)
    print(f"replay n={n} orth={orth:.3e} resid={resid:.3e} ({time.time()-t0:.0f} s)", flush=True)
