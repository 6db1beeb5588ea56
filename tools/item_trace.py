"""Per-work-item device timeline of one factorization (globaltimer stamps,
tqr_set_trace) summarised per kernel kind: busy time, dependency wait,
SM utilisation over time.  Writes a JSON summary (and optional Gantt CSV in
the reference's list-schedule format proc,start,end,kind,i,j,k —
sched.py:36-49)."""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1303_3182_b200 as P  # noqa: E402
from paper_1303_3182_b200 import _lib  # noqa: E402
from paper_1303_3182_b200.engine import Plan  # noqa: E402

KIND = ["GEQRT", "TTQRT", "TSQRT", "UNMQR", "TTMQR", "TSMQR", "PACK", "UNPACK"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--out", default="gpurun_out/item_trace.json")
    ap.add_argument("--gantt", default=None)
    ap.add_argument("--stream", action="store_true", help="trace the streaming host-to-host path")
    ap.add_argument("--family", default=None, choices=["TT", "TS"])
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    if a.family:
        cfg = dict(cfg, family=a.family)
    nb = cfg["nb"]
    p, q = cfg["m"] // nb, cfg["n"] // nb
    b = P.build_tree(p, q, cfg["algo"], family=cfg["family"])
    plan = Plan(b, nb, io=(Plan.IO_IN | Plan.IO_OUT) if a.stream else 0)
    A = torch.from_numpy(bench.make_matrix(cfg))
    tiles, tg, te = plan.alloc()
    if a.stream:
        A = A.pin_memory()
        R = torch.zeros((plan.n, plan.n), dtype=torch.float64).pin_memory()
        bufs = plan.stream_buffers()
        tiles, tg, te = bufs.tiles, bufs.tg, bufs.te
        run = lambda: plan.factor_stream(A, R, bufs)  # noqa: E731
        # raw pinned H2D bandwidth for reference
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        bufs.stage.copy_(A, non_blocking=True)
        ev[1].record()
        torch.cuda.synchronize()
        h2d_ms = ev[0].elapsed_time(ev[1])
    else:
        A = A.cuda()
        run = lambda: (plan.pack(A, tiles), plan.factor(tiles, tg, te))  # noqa: E731
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    n = plan.info.n_items
    tr = torch.zeros(4 * n + 64, dtype=torch.int64, device="cuda")
    _lib.lib().tqr_set_trace(C.c_void_p(tr.data_ptr()))
    import time
    t_w = time.perf_counter()
    run()
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - t_w) * 1e3
    _lib.lib().tqr_set_trace(None)
    trc = tr.cpu().numpy()
    t = trc[:4 * n].reshape(n, 4)
    prof = trc[4 * n:]
    items = np.empty((n, 7), dtype=np.int32)
    _lib.check(_lib.lib().tqr_plan_items(plan._h, _lib.ptr_i32(items)))
    t0 = t[:, 0].min()
    deq, rdy, end, sm = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, t[:, 3]
    total = end.max()
    out = {"config": a.config, "items": int(n), "makespan_us": float(total),
           "gflops": plan.flops / (total * 1e-6) / 1e9, "per_kind": {}}
    if a.stream:
        out["wall_ms"] = wall_ms
        out["h2d_full_ms"] = h2d_ms
        pk = items[:, 0] == 6
        upk = items[:, 0] == 7
        out["pack_last_ready_us"] = float(rdy[pk].max())
        out["pack_ready_deciles_us"] = [round(float(x), 1) for x in np.percentile(rdy[pk], np.arange(0, 101, 10))]
        cmp_ = ~(pk | upk)
        out["compute_first_start_us"] = float(rdy[cmp_].min())
        out["compute_last_end_us"] = float(end[cmp_].max())
        out["unpack_last_end_us"] = float(end[upk].max())
        # completion time of each tile row of R and the modeled D2H queue
        rows_done = np.zeros(plan.q)
        for r in np.nonzero(upk)[0]:
            ii = items[r, 2] - 1
            rows_done[ii] = max(rows_done[ii], end[r])
        fin = 0.0
        for ii in range(plan.q):
            fin = max(fin, rows_done[ii]) + (plan.q - ii) * nb * nb * 8 / 50e9 * 1e6
        out["r_rows_done_us"] = [round(float(x)) for x in rows_done]
        out["modeled_copy_out_end_us"] = fin
        # SM busy (compute kinds only) in 5% bins
        bins = np.linspace(0, end.max(), 21)
        out["compute_busy_by_5pct"] = [round(float(np.clip(np.minimum(end[cmp_], hi) - np.maximum(rdy[cmp_], lo), 0,
                                                           None).sum() / ((hi - lo) * (int(sm.max()) + 1))), 3)
                                       for lo, hi in zip(bins[:-1], bins[1:])]
    for kd in range(8):
        msk = items[:, 0] == kd
        if not msk.any():
            continue
        dur = end[msk] - rdy[msk]
        wait = rdy[msk] - deq[msk]
        out["per_kind"][KIND[kd]] = {"n": int(msk.sum()), "mean_us": float(dur.mean()), "p50_us": float(np.median(dur)),
                                     "p90_us": float(np.percentile(dur, 90)), "sum_ms": float(dur.sum() / 1e3),
                                     "mean_wait_us": float(wait.mean()), "sum_wait_ms": float(wait.sum() / 1e3)}
    names = ["load", "l2_tail", "group_upd", "writeback", "trailing", "gram", "T", "l2_reduce", "l2_D"]
    for md, nm in ((0, "GEQRT"), (1, "TTQRT"), (2, "TSQRT")):
        cnt = int((items[:, 0] == md).sum())
        if cnt:
            out.setdefault("panel_phases_us", {})[nm] = {names[k]: round(float(prof[md * 16 + k]) / 1e3 / cnt, 2)
                                                        for k in range(len(names))}
    out["early_staging"] = {"staged": int(prof[56]), "not_ready": int(prof[57])}
    nsm = int(sm.max()) + 1
    busy = (end - rdy).sum()
    waits = (rdy - deq).sum()
    out["sm_busy_frac"] = float(busy / (nsm * total))
    out["sm_wait_frac"] = float(waits / (nsm * total))
    # gaps between consecutive items on one SM (dequeue overhead + fence)
    gaps = []
    for s in range(nsm):
        m = sm == s
        o = np.argsort(deq[m])
        st, en = deq[m][o], end[m][o]
        gaps.append((st[1:] - en[:-1]).sum() if len(st) > 1 else 0.0)
    out["sm_gap_frac"] = float(np.sum(gaps) / (nsm * total))
    # active items over time (10 bins)
    bins = np.linspace(0, total, 11)
    act = []
    for lo, hi in zip(bins[:-1], bins[1:]):
        ov = np.clip(np.minimum(end, hi) - np.maximum(rdy, lo), 0, None).sum()
        act.append(round(float(ov / ((hi - lo) * nsm)), 3))
    out["busy_by_decile"] = act
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))
    if a.gantt:
        with open(a.gantt, "w") as fh:
            fh.write("proc,start,end,kind,i,j,k\n")
            for r in range(n):
                fh.write(f"{sm[r]},{rdy[r]:.3f},{end[r]:.3f},{KIND[items[r, 0]]},{items[r, 2]},{items[r, 5]},{items[r, 4]}\n")


if __name__ == "__main__":
    main()
