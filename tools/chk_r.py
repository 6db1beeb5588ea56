"""Debug: R of the tiled QR vs cuSOLVER for a few sizes (rel. error)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_3182_b200.engine import tiled_qr

sizes = [int(x) for x in os.environ.get("SIZES", "2048,4096").split(",")]
for m in sizes:
    A = np.random.default_rng(2).standard_normal((m, m))
    At = torch.from_numpy(A).cuda()
    res = tiled_qr(At, nb=256, algo=os.environ.get("ALGO", "greedy"))
    R = res.R()
    Rref = torch.linalg.qr(At, mode="r")[1]
    s1 = torch.sign(torch.diagonal(R)); s2 = torch.sign(torch.diagonal(Rref))
    err = (torch.linalg.norm(torch.nan_to_num(R) * s1[:, None] - Rref * s2[:, None]) / torch.linalg.norm(At)).item()
    print(f"size={m} grid={os.environ.get('TQR_GRID','148')} flags={os.environ.get('TQR_FLAGS','0')} relerr={err:.3e}", flush=True)
