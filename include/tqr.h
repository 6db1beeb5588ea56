/* tqr.h — C ABI of the B200-native tiled QR engine (libtqr.so).
 *
 * The reference (`tiledag`, pkg/src/tiledag) is a pure-Python package with no
 * FFI; its drop-in surface is the Python API re-exported by
 * pkg/src/tiledag/__init__.py:16-24.  Each entry point below replaces one
 * reference function on the hot path (cited per declaration); the Python
 * package paper_1303_3182_b200 binds them with ctypes and keeps the
 * reference signatures unchanged.  Numeric entry points have no reference
 * counterpart (the reference executes no kernels, pkg/README.md:11-12) and
 * extend the same API with A=/nb=/ib=.
 *
 * Conventions: rows/columns of tiles are 1-based like the reference
 * (qr.py:11).  Elimination entries are int32 quadruples (i, piv, k, step).
 * Every function returns 0 on success or a negative TQR_E* status; the
 * message is available from tqr_last_error() (thread-local).  Device
 * pointers are plain CUDA device addresses owned by the caller; `stream` is
 * a cudaStream_t passed as void*.  Plans are immutable after creation and
 * may be launched concurrently on several streams (per-launch scratch slots).
 */
#ifndef TQR_H
#define TQR_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TQR_OK 0
#define TQR_EVALUE (-1)  /* bad input; Python raises ValueError(msg)           */
#define TQR_EKEY (-2)    /* missing state; Python raises KeyError(msg)         */
#define TQR_EASSERT (-3) /* internal invariant; Python raises AssertionError   */
#define TQR_EOTHER (-4)  /* anything else; Python raises RuntimeError          */
#define TQR_ECUDA (-5)   /* CUDA runtime failure; Python raises RuntimeError   */
#define TQR_NO_BS INT32_MIN /* "bs=None" for tqr_build_tree                    */

enum tqr_kind { TQR_GEQRT = 0, TQR_TTQRT = 1, TQR_TSQRT = 2, TQR_UNMQR = 3, TQR_TTMQR = 4, TQR_TSMQR = 5 };

const char* tqr_last_error(void);
int tqr_abi_version(void);

/* ---------------- schedule compiler (host, bit-exact with the reference) -- */

/* coarse_schedule(p, q, algo)            qr.py:279-297
 * steps: p*q int32, index (i-1)*q+(k-1), 0 where no tile is zeroed.
 * elim: 4*cap int32.  *n_out = number of entries, *x_out = table.x.       */
int tqr_coarse_schedule(int p, int q, const char* algo, int32_t* steps, int32_t* elim, int64_t cap,
                        int64_t* n_out, int32_t* x_out);
/* plasmatree_list(p, q, bs) / binary_tree_list (bs=1)   qr.py:336-366      */
int tqr_plasmatree_list(int p, int q, int bs, int32_t* elim, int64_t cap, int64_t* n_out);
/* EliminationList.validate()  qr.py:56-83.  Returns 0 valid, 1 invalid with
 * the reference's ValueError text in msg.                                  */
int tqr_elim_validate(int p, int q, const int32_t* elim, int64_t n, char* msg, int64_t msg_cap);
/* EliminationList.with_steps()  qr.py:118-127                               */
int tqr_elim_with_steps(const int32_t* elim, int64_t n, int32_t* out);
/* EliminationList.normalized()  qr.py:85-116                                */
int tqr_elim_normalized(int p, int q, const int32_t* elim, int64_t n, int32_t* out);

typedef struct tqr_build tqr_build;
typedef struct {
  int32_t p, q, family_ts;
  int64_t cp, total_weight;
  int64_t counts[6]; /* by enum tqr_kind */
  int64_t n_elim, n_trace, n_zeroed, n_updates;
} tqr_build_info;

/* build_tree(p, q, algo, family, bs, grasap_i, weights, keep_trace,
 *            record_updates)   qr.py:622-649.  weights6: by enum tqr_kind,
 * -1 = kind missing from the model, NULL = WeightModel.qr_tt()
 * (taskgraph.py:92-95).                                                     */
int tqr_build_tree(int p, int q, const char* algo, int family_ts, int bs, int grasap_i, const int64_t* weights6,
                   int keep_trace, int record_updates, tqr_build** out);
/* tiled_build(elim, family, weights, keep_trace, record_updates, validate)
 * qr.py:535-540                                                             */
int tqr_tiled_build(int p, int q, const int32_t* elim, int64_t n, int family_ts, const int64_t* weights6,
                    int keep_trace, int record_updates, int validate, tqr_build** out);
/* QrBuild attributes (qr.py:392-408)                                        */
int tqr_build_get_info(const tqr_build* b, tqr_build_info* out);
int tqr_build_get_elim(const tqr_build* b, int32_t* out4);
/* zeroed: (i, k, finish) triples in first-zeroing order                     */
int tqr_build_get_zeroed(const tqr_build* b, int64_t* out3);
/* trace: kind, indices (4 per task, -1 padded), ASAP finish                 */
int tqr_build_get_trace(const tqr_build* b, int8_t* kind, int32_t* idx4, int64_t* fin);
/* record_updates: (i, k, j, finish) per TTMQR in trace order                */
int tqr_build_get_updates(const tqr_build* b, int64_t* out4);
/* build_from_trace edges (taskgraph.py:262-322): (u, v, cause) with cause
 * 0 RAW, 1 WAR, 2 WAW.  Call with uvc=NULL to get *n_out.                   */
int tqr_build_hazard_edges(tqr_build* b, int32_t* uvc, int64_t cap, int64_t* n_out);
/* A build holding an explicit kernel trace (kinds + 1-based indices as in
 * tqr_build_get_trace), e.g. the cross-shard R merge of the tall-skinny
 * path; only the trace is meaningful (no ASAP times).  Feed to
 * tqr_plan_create like any build.                                          */
int tqr_trace_build(int p, int q, const int8_t* kind, const int32_t* idx4, int64_t n, tqr_build** out);
void tqr_build_free(tqr_build* b);

/* ---------------- numeric engine (CUDA, sm_100a) ------------------------- */

typedef struct tqr_plan tqr_plan;
typedef struct {
  int32_t p, q, nb, ib, slab, family_ts;
  int64_t n_tasks, n_items, n_preds;
  int64_t tg_stride, te_stride; /* doubles per (i,k) T slot                   */
  double flops_alg;             /* 2 n^2 (m - n/3), qr.py:663-667 x nb^3/3  */
} tqr_plan_info;

/* Compile a build (keep_trace=1) into a static device schedule: the trace's
 * kernels split into column slabs, hazard edges (taskgraph.py:262-322)
 * refined to slab granularity, items ordered by weighted ASAP start.       */
int tqr_plan_create(const tqr_build* b, int nb, int ib, tqr_plan** out);
/* Same, with streaming I/O work items in the device schedule (io bit 0:
 * PACK items read the row-major input as its tile rows arrive; bit 1:
 * UNPACK items write each finished R tile to row-major (host-mapped) memory
 * as soon as it is final).  Run with tqr_factor_io.                        */
int tqr_plan_create_io(const tqr_build* b, int nb, int ib, int io, tqr_plan** out);
int tqr_plan_get_info(const tqr_plan* plan, tqr_plan_info* out);
void tqr_plan_free(tqr_plan* plan);

/* Row-major (or column-major) m x n matrix -> tile-major p x q tiles of
 * nb x nb, column-major inside a tile; tiles of one tile column contiguous. */
int tqr_pack(const double* A, int64_t lda, int row_major, double* tiles, int p, int q, int nb, void* stream);
int tqr_unpack(const double* tiles, int p, int q, int nb, double* A, int64_t lda, int row_major, void* stream);
/* Upper-triangular R (n x n, n = q*nb) from the factored tiles.            */
int tqr_extract_r(const double* tiles, int p, int q, int nb, double* R, int64_t ldr, int row_major, void* stream);
/* In-place tiled QR: run the plan's kernels (GEQRT, UNMQR, TTQRT, TTMQR,
 * TSQRT, TSMQR) on `tiles`; writes T factors into tg/te (tg_stride /
 * te_stride doubles per tile).  Asynchronous on `stream`.                  */
int tqr_factor(tqr_plan* plan, double* tiles, double* tg, double* te, void* stream);
/* Streaming factorization: a_src = row-major m x n input staging buffer in
 * device memory, filled asynchronously by the caller one arrival unit at a
 * time (tqr_plan_arrival_units: a block of tile rows of one tile column),
 * each unit u followed by setting arrive[u] != 0 on the same copy stream
 * (e.g. cuStreamWriteValue32); arrive[] (n_units ints) must be zero at launch.
 * r_dst = row-major n x n R (device-accessible), strictly-lower part outside
 * the diagonal tiles left untouched.  r_ready (optional, q ints, zero at
 * launch): r_ready[i] counts the tiles of R's tile row i+1 already written,
 * complete at q-i; a copy stream can wait on it (cuStreamWaitValue32 GEQ). */
int tqr_factor_io(tqr_plan* plan, const double* a_src, int64_t lda, const int* arrive, double* tiles, double* tg,
                  double* te, double* r_dst, int64_t ldr, int* r_ready, void* stream);
/* Host-to-host QR (plan made with io = 3): pinned row-major A (lda_h) in,
 * pinned row-major R (ldr_h) out, every transfer overlapped with the
 * factorization.  With io = 1 only A streams in (r_host, r_dev, r_ready may
 * be NULL; the factored tiles stay in `tiles`).  Enqueues on `stream` the executor, on `copy_in` the
 * nb-column blocks of A (one 2D copy each, in tqr_plan_arrival_units order) each
 * followed by its arrival flag, and on `copy_out` one wait + copy per tile
 * row of R; returns at once, `stream` completes after all three.  Device
 * scratch: stage (m*n doubles), arrive (q ints), r_dev (n*n doubles),
 * r_ready (q ints).  The
 * strictly-lower part of r_host outside the diagonal tiles is not written.  */
int tqr_qr_host(tqr_plan* plan, const double* a_host, int64_t lda_h, double* r_host, int64_t ldr_h, double* stage,
                int* arrive, double* tiles, double* tg, double* te, double* r_dev, int* r_ready, void* stream,
                void* copy_in, void* copy_out);
/* Input arrival units of an io plan in transfer order: *n_units, and if
 * units3 != NULL, 3 ints per unit: 1-based tile column j, first tile row i0,
 * number of tile rows.  A unit's flag is arrive[(j-1)*nch + (i0-1)/cr] with
 * cr the chunk height (units3[2] of the first unit) and nch = ceil(p/cr).   */
int tqr_plan_arrival_units(const tqr_plan* plan, int32_t* n_units, int32_t* units3);
/* C <- Q C (trans=0) or Q^T C (trans=1) for C stored as p x c_cols tiles,
 * replaying the trace's reflectors (forward for Q^T, reverse for Q).      */
int tqr_apply_q(tqr_plan* plan, int trans, const double* tiles, const double* tg, const double* te,
                double* c_tiles, int c_cols, void* stream);
/* Diagnostics: record {t_dequeue, t_ready, t_end, smid} (globaltimer ns) per
 * work item of the following tqr_factor/tqr_apply_q calls into trace_dev
 * (4*n_items uint64; NULL disables); tqr_plan_items lists the items
 * (kind, slab, i, piv, k, j, n_preds) in device order.  Gantt export as in
 * the reference's list-schedule CSV (sched.py:36-49).                     */
int tqr_set_trace(void* trace_dev);
int tqr_plan_items(const tqr_plan* plan, int32_t* out7);
/* Device-side FP64 peak probe (DMMA.8x8x4 loop on every SM), TFLOP/s.      */
int tqr_fp64_peak(double* tflops_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TQR_H */
