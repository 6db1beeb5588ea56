"""H2D arrival probe: per-row-block completion times of the pinned input
copy, alone and while the executor runs a device-resident factorization."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1303_3182_b200 as P  # noqa: E402
from paper_1303_3182_b200.engine import Plan  # noqa: E402


def rows(A_pin, stage, nb, s):
    p = A_pin.shape[0] // nb
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(p + 1)]
    with torch.cuda.stream(s):
        ev[0].record(s)
        for i in range(p):
            stage[i * nb:(i + 1) * nb].copy_(A_pin[i * nb:(i + 1) * nb], non_blocking=True)
            ev[i + 1].record(s)
    return ev


def cols(A_pin, stage, nb, s):
    q = A_pin.shape[1] // nb
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(q + 1)]
    with torch.cuda.stream(s):
        ev[0].record(s)
        for j in range(q):
            stage[:, j * nb:(j + 1) * nb].copy_(A_pin[:, j * nb:(j + 1) * nb], non_blocking=True)
            ev[j + 1].record(s)
    return ev


def main():
    cfg = bench.CONFIGS["c3"]
    nb = cfg["nb"]
    p, q = cfg["m"] // nb, cfg["n"] // nb
    A_pin = torch.from_numpy(bench.make_matrix(cfg)).pin_memory()
    stage = torch.empty(A_pin.shape, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    out = {}
    for rep in range(2):
        ev = rows(A_pin, stage, nb, s)
        torch.cuda.synchronize()
    out["alone_ms"] = round(ev[0].elapsed_time(ev[-1]), 2)
    for rep in range(2):
        ev = cols(A_pin, stage, nb, s)
        torch.cuda.synchronize()
    out["cols_alone_ms"] = round(ev[0].elapsed_time(ev[-1]), 2)
    assert torch.equal(stage.cpu(), A_pin)
    for w in (2, 4, 8, 16, 32):
        for rep in range(2):
            ev = cols(A_pin, stage, nb * w, s)
            torch.cuda.synchronize()
        out[f"cols_w{w}_ms"] = [round(ev[0].elapsed_time(e), 2) for e in ev[1:]]
    plan = Plan(P.build_tree(p, q, "greedy"), nb)
    tiles, tg, te = plan.alloc()
    A = A_pin.cuda()
    plan.pack(A, tiles)
    plan.factor(tiles, tg, te)
    torch.cuda.synchronize()
    plan.pack(A, tiles)
    k0 = torch.cuda.Event(enable_timing=True)
    k1 = torch.cuda.Event(enable_timing=True)
    k0.record()
    plan.factor(tiles, tg, te)
    k1.record()
    ev = rows(A_pin, stage, nb, s)
    torch.cuda.synchronize()
    out["with_kernel_ms"] = round(ev[0].elapsed_time(ev[-1]), 2)
    out["kernel_ms"] = k0.elapsed_time(k1)
    # D2H of R rows alone
    R = torch.zeros((cfg["n"], cfg["n"]), dtype=torch.float64).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    R.copy_(stage[:cfg["n"]], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    out["d2h_full_ms"] = e0.elapsed_time(e1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
