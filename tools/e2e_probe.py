"""e2e (tiled_qr_host) timing probe at C3: warm calls with a reused plan and
buffers, before and after one cold call through the plan cache."""
import os, sys, time, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_3182_b200 as P
from paper_1303_3182_b200.engine import Plan, tiled_qr_host

cfg = bench.CONFIGS["c3"]
nb = cfg["nb"]; p, q = cfg["m"] // nb, cfg["n"] // nb
A_host = bench.make_matrix(cfg)
A_pin = torch.from_numpy(A_host).pin_memory()
R_pin = torch.zeros((cfg["n"], cfg["n"]), dtype=torch.float64).pin_memory()
plan_io = Plan(P.build_tree(p, q, "greedy"), nb, io=Plan.IO_IN | Plan.IO_OUT)
bufs = plan_io.stream_buffers()

def warm(tag, n=3):
    tiled_qr_host(A_pin, R_pin, plan=plan_io, buffers=bufs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(n):
        tiled_qr_host(A_pin, R_pin, plan=plan_io, buffers=bufs)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({tag: {"event_ms": e0.elapsed_time(e1) / n, "wall_ms": (time.perf_counter() - t0) * 1e3 / n}}), flush=True)

warm("before_cold")
t0 = time.perf_counter()
tiled_qr_host(A_pin, R_pin, nb=nb, algo="greedy")
torch.cuda.synchronize()
print(json.dumps({"cold_ms": (time.perf_counter() - t0) * 1e3}), flush=True)
warm("after_cold")
os.environ["TQR_IO_DEBUG"] = "1"
warm("debug", 1)
