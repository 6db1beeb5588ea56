"""Orthogonality ||Q^T Q - I||_F of our Q vs cuSOLVER's (same fp64 check)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_3182_b200.engine import tiled_qr

for n in [int(x) for x in os.environ.get("SIZES", "8192,16384").split(",")]:
    A = np.random.default_rng(2).standard_normal((n, n))
    At = torch.from_numpy(A).cuda()
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    res = tiled_qr(At, nb=256, algo="greedy")
    Q = res.Q()
    R = res.R()
    o1 = torch.linalg.norm(Q.T @ Q - I).item()
    r1 = (torch.linalg.norm(At - Q @ R) / torch.linalg.norm(At)).item()
    del Q, R, res
    Qc, Rc = torch.linalg.qr(At)
    o2 = torch.linalg.norm(Qc.T @ Qc - I).item()
    r2 = (torch.linalg.norm(At - Qc @ Rc) / torch.linalg.norm(At)).item()
    print(f"n={n} ours: orth={o1:.3e} resid={r1:.3e}   cusolver: orth={o2:.3e} resid={r2:.3e}", flush=True)
