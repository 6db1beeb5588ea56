"""The thesis' own experiment grid on one B200 (PAPER.md
:2631-2635): m = 8000, n = 200 q for q = 1, 2, 4, 5, 10, 20, 40, double
precision, Greedy / Fibonacci / PlasmaTree (best BS of a small sweep) with TT
kernels.  The thesis used nb = 200 tiles on a 48-core Opteron; here the same
matrices are zero-padded to whole tiles of nb = 128 and 256 (tiled_qr pads),
and GFLOP/s counts the unpadded 2n^2(m - n/3).  Device-resident A, CUDA
events around tiled_qr's pack + factorization, after warm-up.  Prints one
JSON object (the published values beside ours)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1303_3182_b200 as P  # noqa: E402
from paper_1303_3182_b200.engine import Plan  # noqa: E402

# BASELINE.md §1, GFLOP/s, double
PUBLISHED = {
    "greedy": [36.936, 58.509, 103.267, 115.306, 153.518, 170.873, 184.522],
    "plasmatree": [37.502, 52.718, 90.794, 100.554, 145.820, 171.827, 182.816],
    "fibonacci": [26.561, 49.487, 100.144, 115.002, 152.009, 170.478, 180.299],
}
QS = [1, 2, 4, 5, 10, 20, 40]


def run(A, nb, algo, bs, steps=5, warmup=2):
    m, n = A.shape
    p, q = -(-m // nb), -(-n // nb)
    plan = Plan(P.build_tree(p, q, algo, bs=bs), nb)
    Ap = torch.zeros((p * nb, q * nb), dtype=torch.float64, device="cuda")
    Ap[:m, :n] = A
    tiles, tg, te = plan.alloc()

    def step():
        plan.pack(Ap, tiles)
        plan.factor(tiles, tg, te)

    for _ in range(warmup):
        step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return ms, 2.0 * n * n * (m - n / 3.0) / (ms * 1e-3) / 1e9


def main():
    out = {"m": 8000, "qs": QS, "nb_thesis": 200, "published_gflops": PUBLISHED, "b200": {}}
    rng = np.random.default_rng(7)
    A_full = torch.from_numpy(rng.standard_normal((8000, 8000))).cuda()
    for algo in ("greedy", "fibonacci", "plasmatree"):
        rows = []
        for q in QS:
            A = A_full[:, :200 * q]
            best = None
            for nb in (128, 256):
                p_t = -(-8000 // nb)
                q_t = -(-200 * q // nb)
                bss = [None] if algo != "plasmatree" else sorted({b for b in (1, 2, 4, 8, 16, p_t) if b <= p_t})
                for bs in bss:
                    ms, gf = run(A, nb, algo, bs)
                    rec = {"nb": nb, "bs": bs, "tiles": f"{p_t}x{q_t}", "ms": round(ms, 3), "gflops": round(gf, 1)}
                    if best is None or gf > best["gflops"]:
                        best = rec
            best["q"] = q
            best["n"] = 200 * q
            rows.append(best)
            print(json.dumps({algo: best}), file=sys.stderr, flush=True)
        out["b200"][algo] = rows
    print(json.dumps(out))


if __name__ == "__main__":
    main()
