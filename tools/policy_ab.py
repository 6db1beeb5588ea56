"""Executor dequeue policy A/B: the plan's own choice (look-ahead dequeue on
for throughput-bound schedules, off for critical-path-bound ones) against
both forced settings (TQR_FLAGS=0 / 4), on C3, C4, the C5 G=8 shard and C1."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_3182_b200 as P
from paper_1303_3182_b200.engine import Plan

def timed(plan, A, reps):
    tiles, tg, te = plan.alloc()
    for _ in range(2):
        plan.pack(A, tiles); plan.factor(tiles, tg, te)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        plan.pack(A, tiles); plan.factor(tiles, tg, te)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

out = {}
for name, rows, reps in (("c1", None, 20), ("c4", None, 5), ("c5_shard_g8", 1024 * 256, 3), ("c3", None, 2)):
    cfg = bench.CONFIGS[name.split("_")[0]]
    nb = cfg["nb"]
    A = torch.from_numpy(bench.make_matrix(cfg, rows=rows) if rows else bench.make_matrix(cfg)).cuda()
    p, q = A.shape[0] // nb, A.shape[1] // nb
    plan = Plan(P.build_tree(p, q, cfg["algo"]), nb)
    rec = {}
    for tag, fl in (("policy", None), ("lookahead", "0"), ("no_lookahead", "4")):
        if fl is None:
            os.environ.pop("TQR_FLAGS", None)
        else:
            os.environ["TQR_FLAGS"] = fl
        rec[tag] = round(timed(plan, A, reps), 3)
    os.environ.pop("TQR_FLAGS", None)
    out[name] = rec
    print(json.dumps({name: rec}), flush=True)
    del A, plan
    torch.cuda.empty_cache()
