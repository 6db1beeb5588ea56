"""C5 multi-GPU projection from one GPU (this run has one B200): time the
per-rank pieces of dist.tall_skinny_qr — the local Greedy factorization of
p/G tile rows (what every rank does concurrently) and one binary R merge
(what the receiving rank of each of the log2 G rounds does) — on the same
device, and project T(G) = local(G) + log2(G) * (merge + R transfer at the
NVLink p2p rate), and for the gather merge T(G) = local(G) + one merge of
G R blocks + one transfer.  Prints one JSON line.  Not a multi-GPU measurement: the
driver's `bench.py --gpus N` runs are."""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1303_3182_b200 import dist  # noqa: E402


def timed(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    cfg = bench.CONFIGS["c5"]
    nb, m, n = cfg["nb"], cfg["m"], cfg["n"]
    p, q = m // nb, n // nb
    dev = torch.device("cuda", 0)
    flops = 2.0 * n * n * (m - n / 3.0)
    nvlink_gbs = float(os.environ.get("TQR_P2P_GBS", "700"))  # assumed p2p send/recv rate (not measured here)
    out = {"what": "C5 scaling projection from single-GPU timings of the per-rank pieces", "nvlink_p2p_gbs_assumed": nvlink_gbs,
           "G": {}}
    t1 = None
    for G in (1, 2, 4, 8):
        P = p // G
        A = torch.from_numpy(bench.make_matrix(cfg, rows=P * nb, row0=0)).to(dev)
        be = dist.GpuBackend(P, q, nb, dev)
        loc = timed(lambda: be.factor_local(A), 3)
        r_a = be.factor_local(A).clone()
        r_b = r_a.clone()
        mer = timed(lambda: be.merge(r_a.copy_(r_b), r_b), 5) if G > 1 else 0.0
        rs = [r_b.clone() for _ in range(G)]
        gat = timed(lambda: be.merge_many([rs[0].copy_(r_b)] + rs[1:]), 5) if G > 1 else 0.0
        xfer = q * (q + 1) // 2 * nb * nb * 8 / (nvlink_gbs * 1e9) * 1e3  # upper block triangle
        rounds = int(math.log2(G))
        tg = loc + rounds * (mer + xfer)
        tgg = loc + (gat + xfer if G > 1 else 0.0)  # the G-1 sends into rank 0 overlap
        if G == 1:
            t1 = tg
        out["G"][G] = {"local_ms": round(loc, 3), "binary_merge_ms": round(mer, 3), "gather_merge_ms": round(gat, 3),
                       "xfer_ms": round(xfer, 3), "rounds": rounds,
                       "projected_ms_binary": round(tg, 3), "projected_ms_gather": round(tgg, 3),
                       "projected_gflops_gather": round(flops / (tgg * 1e-3) / 1e9, 1),
                       "projected_efficiency_binary": round(t1 / (G * tg), 4),
                       "projected_efficiency_gather": round(t1 / (G * tgg), 4)}
        del A, be
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
