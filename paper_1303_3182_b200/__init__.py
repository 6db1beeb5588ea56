"""B200-native tiled QR engine with the reference `tiledag` QR API.

Schedule side (bit-exact with pkg/src/tiledag/qr.py, via the C++ compiler in
libtqr.so): coarse_schedule, build_tree, tiled_build, asap/grasap builders,
elimination lists, coarse tables, closed forms — re-exported under the
reference's names (pkg/src/tiledag/__init__.py:16-24).

Numeric side (no reference counterpart; hand-written sm_100a kernels):
tiled_qr / TiledQR in engine.py, multi-GPU tall-skinny in dist.py.
"""
from .taskgraph import (  # noqa: F401
    ALL_KINDS, BARRIER, GEQRT, TSMQR, TSQRT, TTMQR, TTQRT, UNMQR,
    CpAnnotation, Task, TaskGraph, TileRef, WeightModel, annotate_cp,
    asap_times, build_from_trace, t_seq, trace_cp,
)
from .qr import (  # noqa: F401
    CoarseTable, ElimEntry, EliminationList, QrBuild, asap_build, asap_graph,
    binary_tree_list, build_tree, coarse_cp_oracle, coarse_schedule,
    eager_coarse, elim_weight, fibonacci_cp_bounds, fibonacci_x,
    flat_tree_list, flattree_cp_composed, flattree_cp_oracle, grasap_build,
    grasap_graph, plasmatree_list, qr_flops, sk_coarse_closed_form,
    tiled_build, tiled_graph, tiled_translation, total_weight,
    verify_weight, zeroed_table_csv,
)


def __getattr__(name):
    # the numeric engine imports torch lazily so schedule users do not pay for it
    if name in ("tiled_qr", "tiled_qr_host", "TiledQR", "Plan"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
