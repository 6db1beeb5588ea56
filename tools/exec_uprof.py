"""Update-item phase split INSIDE the persistent executor (C3 by default):
builds an instrumented copy of the library (-DTQR_PROF_UPD, separate build
dir and .so) and reports, per update item, the consumer warps' cycles in
load_x / wait for staged V (full mbarrier) / apply / store."""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build_prof", "libtqr_prof.so")
if os.environ.get("TQR_LIB_PATH") != OUT:
    env = dict(os.environ, TQR_EXTRA_NVCC_FLAGS="-DTQR_PROF_UPD", TQR_BUILD_DIR=os.path.join(ROOT, "build_prof"),
               TQR_LIB_OUT=OUT, TQR_LIB_PATH=OUT)
    if not os.path.exists(OUT):
        subprocess.check_call([sys.executable, "-c", "from paper_1303_3182_b200 import _build; _build.build()"],
                              cwd=ROOT, env=env)
    os.execve(sys.executable, [sys.executable] + sys.argv, env)

sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
import paper_1303_3182_b200 as P  # noqa: E402
from paper_1303_3182_b200 import _lib  # noqa: E402
from paper_1303_3182_b200.engine import Plan  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
nb = cfg["nb"]
b = P.build_tree(cfg["m"] // nb, cfg["n"] // nb, cfg["algo"], family=cfg["family"])
plan = Plan(b, nb)
A = torch.from_numpy(bench.make_matrix(cfg)).cuda()
tiles, tg, te = plan.alloc()
L = _lib.lib()
L.tqr_debug_uprof.argtypes = [C.POINTER(C.c_ulonglong)]
h = (C.c_ulonglong * 32)()
for rep in range(2):
    plan.pack(A, tiles)
    torch.cuda.synchronize()
    L.tqr_debug_uprof(h)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    plan.factor(tiles, tg, te)
    ev[1].record()
    torch.cuda.synchronize()
    L.tqr_debug_uprof(h)
ms = ev[0].elapsed_time(ev[1])
names = {8: "load_x(first half)", 2: "apply", 6: "store+tail"}
h[0] = sum(h[16:32])
tot = sum(h[k] for k in names) + h[0]
nwarp_items = 8 * (b.counts["UNMQR"] + b.counts["TTMQR"] + b.counts["TSMQR"]) * (nb // 64)
print(f"factor {ms:.1f} ms; update-item consumer cycles per warp-item: {tot / nwarp_items:.0f}")
for k, nm in names.items():
    print(f"  {nm:22s} {h[k] / tot:.3f}  ({h[k] / nwarp_items:.0f} cyc)")
print("  wait_full", round(h[0] / tot, 3))
ng = 8 * b.counts["UNMQR"] * (nb // 64)
nt = 8 * b.counts["TTMQR"] * (nb // 64)
print("  wait_full per block GE:", [round(h[16 + s] / max(ng, 1)) for s in range(8)])
print("  wait_full per block TT:", [round(h[24 + s] / max(nt, 1)) for s in range(8)])
npw = 4 * (b.counts["UNMQR"] + b.counts["TTMQR"] + b.counts["TSMQR"]) * (nb // 64)
print(f"producer per warp-item: wait empty {h[3] / npw:.0f} cyc, issue staging {h[4] / npw:.0f} cyc, between blocks {h[5] / npw:.0f} cyc")
