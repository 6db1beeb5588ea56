// Kernel tasks of the tiled QR (one CTA of 256 threads per work item):
//   update items  UNMQR / TTMQR / TSMQR on one 64-column slab   (qr.py:431-481)
//   panel items   GEQRT / TTQRT / TSQRT on one tile (pair)      (qr.py:421-471)
// Numerics follow LAPACK dgeqrt/dgemqrt/dtpqrt/dtpmqrt (compact WY with ib-
// blocked T), so V, R and T match the oracle's LAPACK replay.
#pragma once
#include "tqr_device.cuh"

namespace tqrk {

// Shared-memory carve-up (doubles).  Update items: Vs[2] + Ts[2] + pivot rows[2].
// Panel items: top block, staged V/T for the trailing update, Gram column
// store, reduction partials, diagonal-row / s broadcasts, per-column scalars.
template <int NB>
struct Smem {
  static constexpr int VS = NB * IB;  // one staged V block
  static constexpr int TS = IB * IB;
  // update layout
  static constexpr int TOP = IB * WS;  // staged pivot rows of a slab (TT/TS)
  static constexpr int U_V0 = 0, U_V1 = VS, U_T0 = 2 * VS, U_T1 = 2 * VS + TS, U_P0 = 2 * VS + 2 * TS,
                       U_P1 = U_P0 + TOP, U_END = U_P1 + TOP;
  // panel layout
  static constexpr int P_TOP = 0, P_V = TS, P_T = P_V + VS, P_G = P_T + TS, P_PART = P_G + TS;
  static constexpr int P_DROW = P_PART + NW * IB, P_SBUF = P_DROW + IB, P_SC = P_SBUF + IB;
  static constexpr int P_END = P_SC + 3 * IB + 8;
  static constexpr int END = U_END > P_END ? U_END : P_END;
  static constexpr size_t BYTES = size_t(END) * sizeof(double);
};

// After the call lane l holds the warp-wide sum of d[l] (recursive halving).
__device__ __forceinline__ double warp_reduce_scatter32(double (&d)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = lane & off;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const double send = up ? d[i] : d[i + off];
      const double keep = up ? d[i + off] : d[i];
      d[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return d[0];
}

// ---------------------------------------------------------------------------
// update item: apply all ib-blocks of one factor's reflectors to a 64-column
// slab of the target tile(s), slab resident in registers for all blocks.

template <int NB, int MODE>
__device__ __forceinline__ void upd_rows(int b, int& r0, int& r1) {
  if (MODE == GE) {
    r0 = b * IB;
    r1 = NB;
  } else if (MODE == TT) {
    r0 = 0;
    r1 = (b + 1) * IB;
  } else {
    r0 = 0;
    r1 = NB;
  }
}

// Producer side of an update item (the NPW producer warps): stage V_b, T_b and the pivot
// rows of every block into the double buffer, running ahead of the compute
// warps (full/empty mbarriers; `seq` numbers staged blocks CTA-wide).
template <int NB, int MODE, bool TRANST>
__device__ void update_produce(double* sm, const double* __restrict__ vt, const double* __restrict__ tt,
                               const double* topt, int slab, int pw, int lane, unsigned long long* full,
                               unsigned long long* empty, unsigned seq) {
  using S = Smem<NB>;
  constexpr int NBLK = NB / IB;
  const int scol0 = slab * WS;
  for (int s = 0; s < NBLK; ++s) {
    const unsigned q = seq + unsigned(s), buf = q & 1u;
    if (q >= 2) mbar_wait(&empty[buf], ((q >> 1) - 1u) & 1u);
    const int b = TRANST ? s : NBLK - 1 - s;
    int r0, r1;
    upd_rows<NB, MODE>(b, r0, r1);
    pstage_v<NB>(sm + (buf ? S::U_V1 : S::U_V0), vt, b, r0, r1, pw, lane);
    pstage_t(sm + (buf ? S::U_T1 : S::U_T0), tt, b, pw, lane);
    if (MODE != GE) pstage_top<NB>(sm + (buf ? S::U_P1 : S::U_P0), topt, scol0, b * IB, pw, lane);
    mbar_arrive_cpasync(&full[buf]);
  }
}

// Compute side (8 warps): the warp's 8 columns of the slab stay in
// registers while all ib-blocks are applied.
template <int NB, int MODE, bool TRANST>
__device__ void update_consume(double* sm, double* xt, double* topt, int slab, int tid, unsigned long long* full,
                               unsigned long long* empty, unsigned seq) {
  using S = Smem<NB>;
  constexpr int NBLK = NB / IB;
  const int warp = tid >> 5, lane = tid & 31;
  UPROF_DECL;
  const int col0 = slab * WS + warp * 8;
  double x[NB / 8][2];
  load_x<NB>(x, xt + size_t(col0) * NB, 0, NB / 8, lane);
  UPROF_MARK(8);
  for (int s = 0; s < NBLK; ++s) {
    const unsigned q = seq + unsigned(s), buf = q & 1u;
    const int b = TRANST ? s : NBLK - 1 - s;
    mbar_wait(&full[buf], (q >> 1) & 1u);
    UPROF_MARK(0);
    int r0, r1;
    upd_rows<NB, MODE>(b, r0, r1);
    const double* Vs = sm + (buf ? S::U_V1 : S::U_V0);
    const double* Ts = sm + (buf ? S::U_T1 : S::U_T0);
    double* top = (MODE == GE) ? nullptr : topt + size_t(col0) * NB + b * IB;
    const double* top_s = (MODE == GE) ? nullptr : sm + (buf ? S::U_P1 : S::U_P0) + warp * 8 * IB;
    warp_apply<NB, TRANST, MODE>(x, r0 / IB, r1 / IB, Vs, Ts, top, lane, top_s, b);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[buf]);
    UPROF_MARK(2);
  }
  store_x<NB>(x, xt + size_t(col0) * NB, 0, NB / 8, lane);
  UPROF_MARK(6);
}

// ---------------------------------------------------------------------------
// panel item: Householder QR of one tile (GE), of [R_piv; R_i] (TT) or of
// [R_piv; A_i] (TS), ib columns at a time.  Level-2 sweep of a block with
// one panel row per thread held in registers: per column a single 32-wide
// warp reduce-scatter yields the column norm, the dots with the trailing
// columns (the reflector application) and the dots with the previous
// reflectors (the Gram column that builds T) — two CTA barriers per column.
// Then T_b (dlarft recurrence) and the block reflector applied to the
// trailing columns on DMMA.

__device__ __forceinline__ unsigned long long ptimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// prof (optional, diagnostics): ns accumulated per phase
// [0 load, 1 level-2, 2 write-back/stage, 3 T, 4 trailing update] + MODE*8
template <int NB, int MODE>
__device__ void panel_item(double* sm, double* at /*GE: tile; TT/TS: bottom tile (i,k)*/,
                           double* rt /*TT/TS: pivot tile (piv,k)*/, double* tslot, int tid,
                           unsigned long long* prof = nullptr) {
  unsigned long long tp = (prof && tid == 0) ? ptimer() : 0;
  auto mark = [&](int ph) {
    if (prof && tid == 0) {
      const unsigned long long t2 = ptimer();
      atomicAdd(prof + MODE * 8 + ph, t2 - tp);
      tp = t2;
    }
  };
  using S = Smem<NB>;
  const int warp = tid >> 5, lane = tid & 31;
  double* Ptop = sm + S::P_TOP;  // TT/TS: top block, column-major ld IB
  double* Vs = sm + S::P_V;
  double* Ts = sm + S::P_T;
  double* G = sm + S::P_G;  // G[i + j*IB] = v_i . v_j, i < j
  double* part = sm + S::P_PART;
  double* drow = sm + S::P_DROW;
  double* sbuf = sm + S::P_SBUF;
  double* tau_s = sm + S::P_SC;
  double* scal_s = tau_s + IB;
  double* beta_s = tau_s + 2 * IB;
  const int t = tid;

  for (int b = 0; b < NB / IB; ++b) {
    const int rb0 = b * IB;
    // thread t owns panel row t: GE tile row rb0+t; TT/TS bottom-tile row t
    const int nrows = (MODE == GE) ? NB - rb0 : (MODE == TT ? rb0 + IB : NB);
    const bool own = t < nrows;
    double row[IB];
#pragma unroll
    for (int c = 0; c < IB; ++c) {
      double v = 0.0;
      if (own) {
        if (MODE == GE)
          v = __ldcg(at + (rb0 + t) + size_t(rb0 + c) * NB);
        else if (MODE == TS || t <= rb0 + c)
          v = __ldcg(at + t + size_t(rb0 + c) * NB);
      }
      row[c] = v;
    }
    if (MODE != GE) {
      for (int e = tid; e < IB * IB; e += NT) {
        const int r = e % IB, c = e / IB;
        Ptop[e] = (r <= c) ? __ldcg(rt + (rb0 + r) + size_t(rb0 + c) * NB) : 0.0;
      }
    }
    csync();
    mark(0);
    // ---- level-2 sweep (dgeqr2 / dtpqrt2 semantics, LAPACK dlarfg).  A
    // runtime loop (small code: the unrolled version is I-cache bound); the
    // register row is indexed statically under predicates.
#pragma unroll 1
    for (int j = 0; j < IB; ++j) {
      if (MODE == GE && t == j) {
#pragma unroll
        for (int c = 0; c < IB; ++c) drow[c] = row[c];
      }
      const bool inv = (MODE == GE) ? (own && t > j) : (MODE == TT ? (t <= rb0 + j) : own);
      double xj = 0.0;
#pragma unroll
      for (int c = 0; c < IB; ++c) xj = (c == j) ? row[c] : xj;
      const double x = inv ? xj : 0.0;
      double d[IB];
#pragma unroll
      for (int c = 0; c < IB; ++c) d[c] = x * row[c];
      part[warp * IB + lane] = warp_reduce_scatter32(d, lane);
      csync();
      if (warp == 0) {
        double D = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) D += part[w * IB + lane];
        const double alpha = (MODE == GE) ? drow[j] : Ptop[j + j * IB];
        const double xn2 = __shfl_sync(0xffffffffu, D, j);
        double tau = 0.0, scal = 0.0, beta = alpha;
        if (xn2 != 0.0) {
          beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
          const double rb = 1.0 / beta;
          tau = (beta - alpha) * rb;
          scal = 1.0 / (alpha - beta);
        }
        const double dr = (MODE == GE) ? drow[lane] : Ptop[j + lane * IB];
        if (lane > j) {
          const double sc = tau * (dr + scal * D);
          sbuf[lane] = sc;
          if (MODE != GE) Ptop[j + lane * IB] = dr - sc;
        }
        if (lane < j) G[lane + j * IB] = scal * D + ((MODE == GE) ? dr : 0.0);
        if (MODE != GE && lane == j) Ptop[j + j * IB] = beta;
        if (lane == 0) {
          tau_s[j] = tau;
          scal_s[j] = scal;
          beta_s[j] = beta;
        }
      }
      csync();
      const double tau = tau_s[j];
      if (tau != 0.0) {
        const double scal = scal_s[j];
        if (inv) {
          const double xs = x * scal;
#pragma unroll
          for (int c = 0; c < IB; ++c) {
            if (c > j) row[c] -= sbuf[c] * xs;
            if (c == j) row[c] = xs;
          }
        }
        if (MODE == GE && t == j) {
#pragma unroll
          for (int c = 0; c < IB; ++c)
            if (c > j) row[c] -= sbuf[c];
        }
      }
      if (MODE == GE && t == j) {
        const double bj = beta_s[j];
#pragma unroll
        for (int c = 0; c < IB; ++c)
          if (c == j) row[c] = bj;
      }
    }
    csync();
    mark(1);
    // ---- write the block back to HBM and stage V for the trailing update
    if (MODE == GE) {
      if (own) {
#pragma unroll
        for (int c = 0; c < IB; ++c) {
          at[(rb0 + t) + size_t(rb0 + c) * NB] = row[c];
          Vs[swz(rb0 + t, c)] = (t > c) ? row[c] : (t == c ? 1.0 : 0.0);
        }
      }
    } else {
      if (own) {
#pragma unroll
        for (int c = 0; c < IB; ++c) {
          const bool live = (MODE == TS) || (t <= rb0 + c);
          if (live) at[t + size_t(rb0 + c) * NB] = row[c];
          Vs[swz(t, c)] = live ? row[c] : 0.0;
        }
      }
      for (int e = tid; e < IB * IB; e += NT) {
        const int r = e % IB, c = e / IB;
        if (r <= c) rt[(rb0 + r) + size_t(rb0 + c) * NB] = Ptop[e];
      }
    }
    csync();
    mark(2);
    // ---- T_b by the dlarft recurrence: lane i owns row i of T
    if (warp == 0) {
      const int i = lane;
      double trow[IB];
#pragma unroll
      for (int l = 0; l < IB; ++l) trow[l] = 0.0;
#pragma unroll 1
      for (int j = 0; j < IB; ++j) {
        const double tj = tau_s[j];
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int l = 0; l < IB; ++l)
          if (l >= i && l < j) s4[l & 3] += trow[l] * G[l + j * IB];
        const double v = (i == j) ? tj : (i < j ? -tj * ((s4[0] + s4[1]) + (s4[2] + s4[3])) : 0.0);
#pragma unroll
        for (int l = 0; l < IB; ++l)
          if (l == j) trow[l] = v;
      }
#pragma unroll
      for (int j = 0; j < IB; ++j) {
        Ts[swz(i, j)] = trow[j];
        tslot[i + size_t(rb0 + j) * IB] = trow[j];
      }
    }
    csync();
    mark(3);
    // ---- trailing update of columns rb0+IB .. NB on DMMA, 8 columns per warp
    const int nch = (NB - rb0 - IB) / 8;
    const int g0 = (MODE == GE) ? rb0 / 8 : 0;
    const int g1 = (MODE == TT) ? (rb0 + IB) / 8 : NB / 8;
    for (int ch = warp; ch < nch; ch += NW) {
      const int col = rb0 + IB + ch * 8;
      double x[NB / 8][2];
      load_x<NB>(x, at + size_t(col) * NB, g0, g1, lane);
      double* top = (MODE == GE) ? nullptr : rt + size_t(col) * NB + rb0;
      warp_apply<NB, true, TS>(x, g0 / (IB / 8), g1 / (IB / 8), Vs, Ts, top, lane);
      store_x<NB>(x, at + size_t(col) * NB, g0, g1, lane);
    }
    csync();
    mark(4);
  }
}

}  // namespace tqrk
