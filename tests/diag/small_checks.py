"""Small end-to-end checks (compute-sanitizer is closed on this pool): C1
(nb=64), a 4x3 nb=256 Greedy/TT and a TS case, apply-Q and the streaming
host-to-host path; R against numpy's QR up to row signs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle.replay import row_sign_normalize  # noqa: E402
from paper_1303_3182_b200.engine import tiled_qr, tiled_qr_host  # noqa: E402


def check(p, q, nb, algo, family="TT"):
    A = np.random.default_rng(p * 100 + q).standard_normal((p * nb, q * nb))
    res = tiled_qr(A, nb=nb, algo=algo, family=family)
    R = row_sign_normalize(res.R().cpu().numpy())
    Rr = row_sign_normalize(np.linalg.qr(A, mode="r"))
    err = np.linalg.norm(R - Rr) / np.linalg.norm(A)
    Qt = res.apply_q(torch.from_numpy(A).cuda(), trans=True).cpu().numpy()
    print(f"{p}x{q} nb={nb} {algo}/{family}: R err {err:.2e}, |Q^T A| below R {np.abs(np.tril(Qt[:q*nb], -1)).max():.2e}")
    assert err < 1e-11
    return A


def main():
    check(8, 4, 64, "greedy")
    check(4, 3, 256, "greedy")
    check(4, 2, 256, "flattree", "TS")
    A = np.random.default_rng(5).standard_normal((4 * 256, 3 * 256))
    R_host, res = tiled_qr_host(torch.from_numpy(A), nb=256, algo="greedy")
    assert torch.equal(R_host, res.R().cpu())
    print("streaming ok")


if __name__ == "__main__":
    main()
