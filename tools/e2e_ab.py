"""e2e at C3 for several modeled H2D rates (TQR_H2D_GBS): fresh plan per rate."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_3182_b200 as P
from paper_1303_3182_b200.engine import Plan, tiled_qr_host
cfg = bench.CONFIGS["c3"]; nb = 256
A_pin = torch.from_numpy(bench.make_matrix(cfg)).pin_memory()
R_pin = torch.zeros((16384, 16384), dtype=torch.float64).pin_memory()
b = P.build_tree(64, 64, "greedy")
for gbs in (60, 48, 40, 32):
    os.environ["TQR_H2D_GBS"] = str(gbs)
    plan = Plan(b, nb, io=3)
    bufs = plan.stream_buffers()
    tiled_qr_host(A_pin, R_pin, plan=plan, buffers=bufs)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(4)]
    for a, e in ev:
        a.record(); tiled_qr_host(A_pin, R_pin, plan=plan, buffers=bufs); e.record()
    torch.cuda.synchronize()
    print(json.dumps({gbs: [round(a.elapsed_time(e), 2) for a, e in ev]}), flush=True)
    del plan, bufs
    torch.cuda.empty_cache()
