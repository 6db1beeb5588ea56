// Persistent dataflow executor (device side), shared by the per-(nb, trans)
// translation units tqr_exec_<nb><t|n>.cu so they compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include "sched.hpp"
#include "tqr_tasks.cuh"

using namespace tqrk;

namespace tqrx {

struct Item {
  int8_t kind;
  int8_t slab;
  int16_t pad;
  int32_t i, piv, k, j;
  int32_t pred_lo, pred_n;
};
static_assert(sizeof(Item) == 28, "item layout");

struct ExecParams {
  const Item* items;
  const int32_t* preds;
  int n_items;
  int* done;
  int* queue;
  const double* vtiles;  // reflector source (factored tiles)
  double* tiles;         // tiles the items write (== vtiles when factoring)
  double* tg;
  double* te;
  int p;
  unsigned long long* trace;  // optional: per item {t_dequeue, t_ready, t_end, smid}
  int flags;                  // debug: bit 0 = no early staging
  // streaming I/O (PACK / UNPACK items)
  const double* a_src;  // row-major input staging (device), ld lda
  long long lda;
  const int* arrive;  // per arrival unit (tile column j, row chunk): nonzero once it landed in a_src
  double* r_dst;      // row-major R output (device-accessible), ld ldr
  long long ldr;
  int* r_ready;  // optional: per tile row of R, count of tiles written out
  int acr, anch;  // arrival units: acr tile rows per chunk, anch chunks per tile column
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}

template <int NB>
__device__ __forceinline__ size_t toff(int p, int i, int j) {
  return (size_t(j - 1) * size_t(p) + size_t(i - 1)) * size_t(NB) * NB;
}
template <int NB>
__device__ __forceinline__ size_t soff(int p, int i, int k) {
  return (size_t(k - 1) * size_t(p) + size_t(i - 1)) * size_t(IB) * NB;
}

// L2 prefetch of the tiles the next work item will touch (its data tiles;
// reflector tiles are shared by many items and usually resident).
template <int NB>
__device__ __forceinline__ void prefetch_item(const ExecParams& P, const Item& I) {
  const unsigned tile_bytes = unsigned(NB) * NB * sizeof(double);
  const unsigned slab_bytes = unsigned(WS) * NB * sizeof(double);
  switch (I.kind) {
    case tqr::GEQRT:
      prefetch_l2(P.tiles + toff<NB>(P.p, I.i, I.k), tile_bytes);
      break;
    case tqr::TTQRT:
    case tqr::TSQRT:
      prefetch_l2(P.tiles + toff<NB>(P.p, I.i, I.k), tile_bytes);
      prefetch_l2(P.tiles + toff<NB>(P.p, I.piv, I.k), tile_bytes);
      break;
    case tqr::UNMQR:
      prefetch_l2(P.tiles + toff<NB>(P.p, I.i, I.j) + size_t(I.slab) * WS * NB, slab_bytes);
      break;
    default:
      prefetch_l2(P.tiles + toff<NB>(P.p, I.i, I.j) + size_t(I.slab) * WS * NB, slab_bytes);
      prefetch_l2(P.tiles + toff<NB>(P.p, I.piv, I.j) + size_t(I.slab) * WS * NB, slab_bytes);
      break;
  }
}

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// PACK(i,j): wait until the arrival unit holding tile (i,j) of the row-major
// input has landed (the host's copy stream raises its flag after the copy), then transpose
// tile (i,j) into the tile-major, column-major-tile layout.  32-row chunks
// through padded smem (LD = NB+1: both phases bank-conflict free); the next
// chunk's loads are issued before the current chunk is written out.
template <int NB>
__device__ void pack_item(double* sm, const ExecParams& P, int i, int j, int tid) {
  constexpr int CR = 32, LD = NB + 1, PER = CR * NB / NT;
  if (tid == 0) {
    while (ld_acquire_sys(P.arrive + (j - 1) * P.anch + (i - 1) / P.acr) == 0) __nanosleep(256);
  }
  csync();
  double* dst = P.tiles + toff<NB>(P.p, i, j);
  const double* src = P.a_src + (long long)(i - 1) * NB * P.lda + (long long)(j - 1) * NB;
  const int warp = tid >> 5, lane = tid & 31;
  double v[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = tid + u * NT;
    v[u] = __ldcg(src + (long long)(e / NB) * P.lda + e % NB);
  }
  for (int r0 = 0; r0 < NB; r0 += CR) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * NT;
      sm[(e / NB) * LD + e % NB] = v[u];
    }
    csync();
    if (r0 + CR < NB) {
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int e = tid + u * NT;
        v[u] = __ldcg(src + (long long)(r0 + CR + e / NB) * P.lda + e % NB);
      }
    }
#pragma unroll 8
    for (int c = warp; c < NB; c += NW) __stcg(dst + size_t(c) * NB + r0 + lane, sm[lane * LD + c]);
    csync();
  }
}

// UNPACK(i,j): final R tile (i,j) (j >= i) -> row-major R (upper triangle
// for the diagonal tile, zeros below it); then, if the caller asked for it,
// count the tile in r_ready[i-1] so a copy stream waiting on that counter
// can ship R's tile row i as soon as all q-i+1 of its tiles are out.
template <int NB>
__device__ void unpack_item(double* sm, const ExecParams& P, int i, int j, int tid) {
  constexpr int CR = 32, LD = NB + 1, PER = CR * NB / NT;
  const double* src = P.tiles + toff<NB>(P.p, i, j);
  double* dst = P.r_dst + (long long)(i - 1) * NB * P.ldr + (long long)(j - 1) * NB;
  const int warp = tid >> 5, lane = tid & 31;
  for (int r0 = 0; r0 < NB; r0 += CR) {
    double v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int c = warp + u * NW;
      v[u] = __ldcg(src + size_t(c) * NB + r0 + lane);
      if (i == j && r0 + lane > c) v[u] = 0.0;
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) sm[lane * LD + warp + u * NW] = v[u];
    csync();
#pragma unroll 8
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * NT;
      __stcg(dst + (long long)(r0 + e / NB) * P.ldr + e % NB, sm[(e / NB) * LD + e % NB]);
    }
    csync();
  }
  if (P.r_ready) {
    __threadfence_system();
    csync();
    if (tid == 0) atomicAdd(P.r_ready + (i - 1), 1);
  }
}

__device__ __forceinline__ bool is_update_kind(int k) { return k == tqr::UNMQR || k == tqr::TTMQR || k == tqr::TSMQR; }

// Warp-specialized persistent executor.  Warpgroups 0-1 (8 warps, 232
// registers) run the kernels; warpgroup 2 (40 registers) stages reflector
// blocks for update items (warp 8) and prefetches the next item's tiles into
// L2 (warp 9).  Per item the roles meet at one CTA barrier (item
// finished); the consumers check dependencies on their own barrier and the
// producer publishes completion flags, so neither waits for the other's
// memory fences.
// COMP: apply-Q kernels (update items only, compensated accumulation).
template <int NB, bool TRANST, bool COMP>
__global__ void __launch_bounds__(NTP, 1) exec_kernel(ExecParams P) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_cur, s_nxt;
  __shared__ int s_ready;  // item whose predecessors the producer already acquired (or -1)
  __shared__ __align__(8) unsigned long long bars[4];  // full[2], empty[2]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // each CTA holds one dequeued item ahead (deadlock-free: items are taken in
  // a topological order and an item only waits on lower-numbered ones)
  if (tid == 0) {
    mbar_init(&bars[0], 2 * 32 * NPW);
    mbar_init(&bars[1], 2 * 32 * NPW);
    mbar_init(&bars[2], NW);
    mbar_init(&bars[3], NW);
    s_cur = atomicAdd(P.queue, 1);
    // flags bit 2: no look-ahead dequeue (an item is taken only when the CTA
    // is free: no early staging, but no item held behind a long one either)
    s_nxt = (s_cur < P.n_items && !(P.flags & 4)) ? atomicAdd(P.queue, 1) : P.n_items;
    s_ready = -1;
  }
  bar_all();
  unsigned seq = 0;
  constexpr unsigned NBLK = NB / IB;
  if (warp >= NW) {
    setmaxnreg_dec<40>();
    __shared__ int s_early;  // producer decision: next item's block 0 staged early
    int pre = 0;             // block 0 of the current item is already staged
    const int pw = warp - NW;
    auto produce = [&](const Item& J, int s_begin, int s_end, unsigned sq) {
      const double* vt = P.vtiles + toff<NB>(P.p, J.i, J.k);
      if (J.kind == tqr::UNMQR)
        update_produce<NB, GE, TRANST>(sm, vt, P.tg + soff<NB>(P.p, J.i, J.k), nullptr, J.slab, pw, lane, bars,
                                       bars + 2, sq, s_begin, s_end);
      else if (J.kind == tqr::TTMQR)
        update_produce<NB, TT, TRANST>(sm, vt, P.te + soff<NB>(P.p, J.i, J.k), P.tiles + toff<NB>(P.p, J.piv, J.j),
                                       J.slab, pw, lane, bars, bars + 2, sq, s_begin, s_end);
      else
        update_produce<NB, TS, TRANST>(sm, vt, P.te + soff<NB>(P.p, J.i, J.k), P.tiles + toff<NB>(P.p, J.piv, J.j),
                                       J.slab, pw, lane, bars, bars + 2, sq, s_begin, s_end);
    };
    int it = s_cur, nx = s_nxt;
    for (;;) {
      if (it >= P.n_items) break;
      const Item I = P.items[it];
      if (warp == NW && lane == 0 && nx < P.n_items && !(P.flags & 2)) prefetch_item<NB>(P, P.items[nx]);
      const bool upd = is_update_kind(I.kind);
      if (upd) {
        if (!pre) {
          // not staged early: wait for the item's predecessors here (the
          // consumers check them too, on their own barrier)
          if (tid == NT) {
            for (int t = 0; t < I.pred_n; ++t) {
              const int pr = P.preds[I.pred_lo + t];
              while (ld_acquire(P.done + pr) == 0) __nanosleep(40);
            }
            __threadfence();  // drop stale L1 lines before cp.async.ca reads
          }
          asm volatile("bar.sync 2, 128;\n" ::: "memory");
        }
        produce(I, pre ? 1 : 0, NBLK, seq);
      }
      unsigned seq_next = seq + (upd ? NBLK : 0);
      // stage block 0 of the next update item now if its predecessors are
      // already done (non-blocking; never when it depends on this item)
      pre = 0;
      // (only behind an update item: a panel item uses the same shared memory)
      if (upd && nx < P.n_items && !(P.flags & 1)) {
        const Item J = P.items[nx];
        if (is_update_kind(J.kind)) {
          if (tid == NT) {
            int ok = 1;
            for (int t = 0; t < J.pred_n && ok; ++t) {
              const int pr = P.preds[J.pred_lo + t];
              ok = (pr != it) && ld_acquire(P.done + pr) != 0;
            }
            if (ok) __threadfence();  // drop stale L1 lines before cp.async.ca reads
            s_early = ok;
            // the consumers may skip their own check of nx (read after the
            // item-finished barrier, which orders this acquire before them)
            s_ready = ok ? nx : -1;
            if (P.trace) atomicAdd(P.trace + 4 * size_t(P.n_items) + 56 + (ok ? 0 : 1), 1ull);
          }
          asm volatile("bar.sync 2, 128;\n" ::: "memory");
          pre = s_early;
          if (pre) produce(J, 0, 1, seq_next);
        }
      }
      seq = seq_next;
      bar_all();  // item finished: every consumer store of `it` is issued
      const int done_it = it;
      it = s_cur;
      nx = s_nxt;
      // publish `it` off the consumers' path: the CTA barrier orders their
      // stores before this thread's gpu-scope fence (cumulative), which
      // waits for them to drain; then the release flag
      if (tid == NT) {
        __threadfence();
        st_release(P.done + done_it, 1);
      }
    }
    return;
  }
  setmaxnreg_inc<232>();
  int it = s_cur, nx = s_nxt;
  for (;;) {
    if (it >= P.n_items) break;
    const Item I = P.items[it];
    unsigned long long t_deq = 0;
    if (P.trace && tid == 0) t_deq = gtimer();
    if (s_ready != it) {
      if (warp == 0) {
        for (int t = lane; t < I.pred_n; t += 32) {
          const int pr = P.preds[I.pred_lo + t];
          while (ld_acquire(P.done + pr) == 0) __nanosleep(40);
        }
        __syncwarp();
        __threadfence();  // gpu-scope fence: also drops stale L1 lines
      }
      csync();  // dependencies satisfied (the producer checks them itself)
    }
    unsigned long long t_rdy = 0;
    if (P.trace && tid == 0) t_rdy = gtimer();
    unsigned long long* pprof = P.trace ? P.trace + 4 * size_t(P.n_items) : nullptr;
    switch (I.kind) {
      case tqr::GEQRT:
        if constexpr (TRANST && !COMP)
          panel_run<NB, GE>(sm, P.tiles + toff<NB>(P.p, I.i, I.k), nullptr, P.tg + soff<NB>(P.p, I.i, I.k), tid, pprof);
        break;
      case tqr::TTQRT:
        if constexpr (TRANST && !COMP)
          panel_run<NB, TT>(sm, P.tiles + toff<NB>(P.p, I.i, I.k), P.tiles + toff<NB>(P.p, I.piv, I.k),
                             P.te + soff<NB>(P.p, I.i, I.k), tid, pprof);
        break;
      case tqr::TSQRT:
        if constexpr (TRANST && !COMP)
          panel_run<NB, TS>(sm, P.tiles + toff<NB>(P.p, I.i, I.k), P.tiles + toff<NB>(P.p, I.piv, I.k),
                             P.te + soff<NB>(P.p, I.i, I.k), tid, pprof);
        break;
      case tqr::PACK:
        if constexpr (TRANST && !COMP) pack_item<NB>(sm, P, I.i, I.j, tid);
        break;
      case tqr::UNPACK:
        if constexpr (TRANST && !COMP) unpack_item<NB>(sm, P, I.i, I.j, tid);
        break;
      case tqr::UNMQR:
        update_consume<NB, GE, TRANST, COMP>(sm, P.tiles + toff<NB>(P.p, I.i, I.j), nullptr, I.slab, tid, bars, bars + 2,
                                       seq);
        break;
      case tqr::TTMQR:
        update_consume<NB, TT, TRANST, COMP>(sm, P.tiles + toff<NB>(P.p, I.i, I.j), P.tiles + toff<NB>(P.p, I.piv, I.j),
                                       I.slab, tid, bars, bars + 2, seq);
        break;
      case tqr::TSMQR:
        update_consume<NB, TS, TRANST, COMP>(sm, P.tiles + toff<NB>(P.p, I.i, I.j), P.tiles + toff<NB>(P.p, I.piv, I.j),
                                       I.slab, tid, bars, bars + 2, seq);
        break;
    }
    if (is_update_kind(I.kind)) seq += NBLK;
    // take the item after next now; the producer warpgroup publishes `it`
    // after the barrier (its fence waits for this CTA's stores to drain while
    // the consumers already start the next item)
    if (tid == 0 && P.trace) {
      P.trace[4 * size_t(it)] = t_deq;
      P.trace[4 * size_t(it) + 1] = t_rdy;
      P.trace[4 * size_t(it) + 2] = gtimer();
      P.trace[4 * size_t(it) + 3] = smid();
    }
    if (P.flags & 4) {
      if (tid == 0) {
        s_cur = atomicAdd(P.queue, 1);
        s_nxt = P.n_items;
      }
    } else if (!(P.flags & 8) && nx < P.n_items && s_ready != nx) {
      // opportunistic order: the held item nx was not found ready by the
      // producer; if it still is not, take the next item from the queue and,
      // when that one is ready, run it first (nx stays held).  Deadlock-free:
      // a CTA only ever waits on the earliest item it holds, and the globally
      // earliest unfinished item is always ready.  Predecessors equal to the
      // item just finished count as done (published right after the barrier).
      if (warp == 0) {
        auto ready = [&](int x) {
          const Item X = P.items[x];
          int ok = 1;
          for (int t = lane; t < X.pred_n; t += 32) {
            const int pr = P.preds[X.pred_lo + t];
            if (pr != it && ld_acquire(P.done + pr) == 0) ok = 0;
          }
          // a PACK item is ready once its arrival unit has landed (otherwise
          // the CTA would sit in it waiting for the host copy while ready
          // work queues behind: the modeled arrival times are only a model)
          if (X.kind == tqr::PACK && lane == 0 &&
              ld_acquire_sys(P.arrive + (X.j - 1) * P.anch + (X.i - 1) / P.acr) == 0)
            ok = 0;
          return __all_sync(0xffffffffu, ok) != 0;
        };
        int cur = nx, nxt;
        if (ready(nx)) {
          nxt = __shfl_sync(0xffffffffu, lane == 0 ? atomicAdd(P.queue, 1) : 0, 0);
        } else {
          const int c = __shfl_sync(0xffffffffu, lane == 0 ? atomicAdd(P.queue, 1) : 0, 0);
          if (c < P.n_items && ready(c)) {
            cur = c;
            nxt = nx;
          } else {
            nxt = c;
          }
          if (P.trace && lane == 0) atomicAdd(P.trace + 4 * size_t(P.n_items) + 58 + (cur == c ? 0 : 1), 1ull);
        }
        if (lane == 0) {
          s_cur = cur;
          s_nxt = nxt;
        }
      }
    } else if (tid == 0) {
      s_cur = nx;
      s_nxt = nx < P.n_items ? atomicAdd(P.queue, 1) : P.n_items;
    }
    bar_all();
    it = s_cur;
    nx = s_nxt;
  }
}

extern int g_flags;
extern int g_carveout;  // debug: TQR_CARVEOUT (percent of the unified L1/smem for shared memory)

struct IoBufs {
  const double* a_src = nullptr;
  long long lda = 0;
  const int* arrive = nullptr;
  double* r_dst = nullptr;
  long long ldr = 0;
  int* r_ready = nullptr;
  int acr = 1, anch = 1;
};

struct DevView {
  const Item* items;
  const int32_t* preds;
  int* done;
  int* queue;
  int n_items;
};

template <int NB, bool TRANST, bool COMP>
cudaError_t launch_exec(const DevView& d, const double* vtiles, double* tiles, double* tg, double* te, int p,
                        unsigned long long* trace, int grid, cudaStream_t st, const IoBufs& io);

// specializations live in tqr_exec_<nb><t|n>.cu
#define TQR_DECLARE_LAUNCH(NB, TR, CO)                                                                              \
  template <>                                                                                                      \
  cudaError_t launch_exec<NB, TR, CO>(const DevView& d, const double* vtiles, double* tiles, double* tg, double* te,  \
                                  int p, unsigned long long* trace, int grid, cudaStream_t st, const IoBufs& io);
TQR_DECLARE_LAUNCH(64, true, false)
TQR_DECLARE_LAUNCH(64, true, true)
TQR_DECLARE_LAUNCH(64, false, true)
TQR_DECLARE_LAUNCH(128, true, false)
TQR_DECLARE_LAUNCH(128, true, true)
TQR_DECLARE_LAUNCH(128, false, true)
TQR_DECLARE_LAUNCH(256, true, false)
TQR_DECLARE_LAUNCH(256, true, true)
TQR_DECLARE_LAUNCH(256, false, true)

#define TQR_DEFINE_LAUNCH(NB, TR, CO)                                                                               \
  template <>                                                                                                      \
  cudaError_t launch_exec<NB, TR, CO>(const DevView& d, const double* vtiles, double* tiles, double* tg, double* te,  \
                                  int p, unsigned long long* trace, int grid, cudaStream_t st,                     \
                                  const IoBufs& io) {                                                              \
    auto kern = exec_kernel<NB, TR, CO>;                                                                               \
    const size_t smem = Smem<NB>::BYTES;                                                                           \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));            \
    if (e != cudaSuccess) return e;                                                                                \
    if (g_carveout >= 0) {                                                                                         \
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, g_carveout);                 \
      if (e != cudaSuccess) return e;                                                                              \
    }                                                                                                              \
    ExecParams P{d.items,  d.preds, d.n_items, d.done,  d.queue,  vtiles,   tiles, tg,                              \
                 te,       p,       trace,     g_flags, io.a_src, io.lda, io.arrive, io.r_dst, io.ldr, io.r_ready, io.acr, io.anch};           \
    kern<<<grid, NTP, smem, st>>>(P);                                                                               \
    return cudaGetLastError();                                                                                     \
  }

}  // namespace tqrx
