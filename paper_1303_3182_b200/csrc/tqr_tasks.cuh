// Kernel tasks of the tiled QR (one CTA of 256 threads per work item):
//   update items  UNMQR / TTMQR / TSMQR on one 64-column slab   (qr.py:431-481)
//   panel items   GEQRT / TTQRT / TSQRT on one tile (pair)      (qr.py:421-471)
// Numerics follow LAPACK dgeqrt/dgemqrt/dtpqrt/dtpmqrt (compact WY with ib-
// blocked T), so V, R and T match the oracle's LAPACK replay.
#pragma once
#include "tqr_device.cuh"

namespace tqrk {

// Shared-memory carve-up (doubles), kept small: what is left of the
// unified 256 KB L1/shared memory is L1, which the 8-byte cp.async staging of
// reflector blocks relies on (forcing the largest carveout costs 4 % at C3).
// Update items: Vs[2] + Ts[2] (the pivot rows of TT/TS items are read from
// global memory, in flight during the first GEMM).  Panel items: the stacked
// panel P, Ts, then a region shared by the factorization scratch (Gram, T,
// group-update partials, per-column scalars) and the staged V of the
// trailing update (written after T is staged, dead before the next block).
template <int NB>
struct Smem {
  static constexpr int VS = NB * IB;  // one staged V block
  static constexpr int TS = IB * IB;
  // update layout
  static constexpr int U_V0 = 0, U_V1 = VS, U_T0 = 2 * VS, U_T1 = 2 * VS + TS, U_END = 2 * VS + 2 * TS;
  // panel layout: stacked panel P (column-major, ld PLD = 4 mod 16)
  static constexpr int PLD = NB + IB + 4;
  static constexpr int LDW = IB + 4;
  static constexpr int P_P = 0, P_T = P_P + PLD * IB, P_X = P_T + TS;
  static constexpr int P_V = P_X;  // aliases everything below
  static constexpr int P_G = P_X, P_TT = P_G + TS;
  static constexpr int P_WP = P_TT + TS, P_W = P_WP + NW * 8 * LDW, P_TG = P_W + 8 * LDW;
  static constexpr int P_PART = P_TG + 64, P_DROW = P_PART + 2 * NW * 8, P_SBUF = P_DROW + 16, P_SC = P_SBUF + 8;
  static constexpr int P_SCR_END = P_SC + 3 * IB + 8;
  static constexpr int P_END = (P_V + VS > P_SCR_END) ? P_V + VS : P_SCR_END;
  // look-ahead panel (panel_item_la): the staged V of the trailing update
  // is live while the next block is factored, so only the Gram / T scratch
  // (G, T plain, the Gram halves' overflow) aliases it; the per-warp partial
  // W is sized for the FW factorization warps
  static constexpr int FW = 4;
  static constexpr int L_W = P_T + TS, L_TG = L_W + 8 * LDW, L_PART = L_TG + 64, L_DROW = L_PART + 2 * NW * 8;
  static constexpr int L_SBUF = L_DROW + 16, L_SC = L_SBUF + 8, L_WP = L_SC + 3 * IB + 8;
  static constexpr int L_V = L_WP + FW * 8 * LDW, L_G = L_V + 256, L_TT = L_G + TS;
  static constexpr int L_G1 = L_TT + TS;  // second halves of the Gram units: [pair][hi 64 | lo 64]
  static constexpr int L_END = (L_V + VS > L_G1 + 1280) ? L_V + VS : L_G1 + 1280;
  static_assert(L_V % 2 == 0, "16-byte aligned staging");
  static constexpr int END0 = U_END > P_END ? U_END : P_END;
#ifndef TQR_PANEL_NO_LA
  static constexpr int END = END0 > L_END ? END0 : L_END;
#else
  static constexpr int END = END0;
#endif
  static constexpr size_t BYTES = size_t(END) * sizeof(double);
};

// 1/sqrt(s) and 1/t for s, t in the normal range: MUFU seed + one cubic
// Newton step (~1 ulp; no IEEE special-case branches).
__device__ __forceinline__ double rsqrt_nr(double s) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
  const double e = fma(-s * y, y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}
__device__ __forceinline__ double rcp_nr(double t) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
  const double e = fma(-t, y, 1.0);
  return fma(y, fma(e, e, e), y);
}

// dlarfg's scalars from alpha and xn2 = ||x||^2 (LAPACK dlarfg, with the
// norm supplied): beta = -sign(alpha) sqrt(alpha^2 + xn2), tau = (beta -
// alpha) / beta, scal = 1 / (alpha - beta); xn2 == 0 gives tau = 0, beta =
// alpha.  With r = 1/sqrt(alpha^2 + xn2): tau = 1 + |alpha| r in [1, 2),
// scal = sign(alpha) r / tau, beta = -sign(alpha) (alpha^2 + xn2) r — one
// rsqrt and one reciprocal, MUFU seeds + one cubic Newton step each, no IEEE
// special-case branches (the caller keeps the arguments in the normal range:
// the panel's scaled path); ~1 ulp.  TQR_L2_IEEE_SCALARS: correctly rounded
// sqrt and division (measured 5 % slower level-2: 143.6 vs 136.4 us).
__device__ __forceinline__ void dlarfg_scalars(double alpha, double xn2, double& tau, double& scal, double& beta) {
  tau = 0.0;
  scal = 0.0;
  beta = alpha;
  if (xn2 != 0.0) {
#ifndef TQR_L2_IEEE_SCALARS
    const double sg = copysign(1.0, alpha);
    const double sq = fma(alpha, alpha, xn2);
    const double r = rsqrt_nr(sq);
    tau = fma(fabs(alpha), r, 1.0);
    scal = sg * r * rcp_nr(tau);
    beta = -sg * sq * r;
#else
    beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
    // tau = (beta - alpha) / beta and 1 / (alpha - beta) from one division
    const double am = alpha - beta, rr = 1.0 / (am * beta);
    tau = -(am * am) * rr;
    scal = beta * rr;
#endif
  }
}

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
                               unsigned long long* empty, unsigned seq, int s_begin = 0, int s_end = NB / IB) {
  using S = Smem<NB>;
  constexpr int NBLK = NB / IB;
  const int scol0 = slab * WS;
  UPROF_DECL_V(_pp);
  for (int s = s_begin; s < s_end; ++s) {
    const unsigned q = seq + unsigned(s), buf = q & 1u;
    UPROF_MARK_V(5, _pp);
    if (q >= 2) mbar_wait(&empty[buf], ((q >> 1) - 1u) & 1u);
    UPROF_MARK_V(3, _pp);
    const int b = TRANST ? s : NBLK - 1 - s;
    int r0, r1;
    upd_rows<NB, MODE>(b, r0, r1);
    pstage_v<NB, MODE>(sm + (buf ? S::U_V1 : S::U_V0), vt, b, r0, r1, pw, lane);
    pstage_t(sm + (buf ? S::U_T1 : S::U_T0), tt, b, pw, lane);
    mbar_arrive_cpasync(&full[buf]);  // completion of this thread's copies
    mbar_arrive(&full[buf]);          // release of its direct stores
    UPROF_MARK_V(4, _pp);
  }
}

// Compute side (8 warps): the warp's 8 columns of the slab stay in
// registers while all ib-blocks are applied.
template <int NB, int MODE, bool TRANST, bool COMP = false>
__device__ void update_consume(double* sm, double* xt, double* topt, int slab, int tid, unsigned long long* full,
                               unsigned long long* empty, unsigned seq) {
  using S = Smem<NB>;
  constexpr int NBLK = NB / IB;
  const int warp = tid >> 5, lane = tid & 31;
  UPROF_DECL;
  const int col0 = slab * WS + warp * 8;
  double* const xc = xt + size_t(col0) * NB;
  double x[NB / 8][2];
  // one reflector block: wait for its staged V/T, apply, release the buffer
  auto block = [&](int s, auto rbl, auto rbh, auto pf) {
    const unsigned q = seq + unsigned(s), buf = q & 1u;
    const int b = TRANST ? s : NBLK - 1 - s;
#ifndef TQR_ABL_NOPROD
    mbar_wait(&full[buf], (q >> 1) & 1u);
#endif
    UPROF_MARK((MODE == GE ? 16 : 24) + s);
    int r0, r1;
    upd_rows<NB, MODE>(b, r0, r1);
    const double* Vs = sm + (buf ? S::U_V1 : S::U_V0);
    const double* Ts = sm + (buf ? S::U_T1 : S::U_T0);
    double* top = (MODE == GE) ? nullptr : topt + size_t(col0) * NB + b * IB;
    const double* top_s = nullptr;  // pivot rows straight from global memory
    warp_apply<NB, TRANST, MODE, decltype(rbl)::value, decltype(rbh)::value, decltype(pf), NoMid, COMP>(
        x, r0 / IB, r1 / IB, Vs, Ts, top, lane, top_s, b, pf);
    __syncwarp();
#ifndef TQR_ABL_NOPROD
    if (lane == 0) mbar_arrive(&empty[buf]);
#endif
    UPROF_MARK(2);
  };
  using R0 = std::integral_constant<int, 0>;
  using RH = std::integral_constant<int, NBLK / 2>;
  using RN = std::integral_constant<int, NBLK>;
  constexpr int GH = NB / 16;  // x row groups of the upper half
  if constexpr (TRANST && MODE == TT) {
    // Q^T with an upper-triangular V: block b only reads x rows of blocks
    // <= b, so the lower half of X loads during block 0's DMMAs
    load_x<NB, false>(x, xc, 0, GH, lane);
    UPROF_MARK(8);
    block(0, R0{}, RH{}, XSched<NB, XS_TT_LOAD>{xc, lane});
    for (int s = 1; s < NBLK / 2; ++s) block(s, R0{}, RH{}, NoPf());
    for (int s = NBLK / 2; s < NBLK; ++s) block(s, R0{}, RN{}, NoPf());
    store_x<NB>(x, xc, 0, NB / 8, lane);
  } else if constexpr (TRANST && MODE == GE) {
    // Q^T with a unit-lower V: the lower half of X loads during block 0's
    // first GEMM on the upper half; rows of blocks < b are final once block b
    // starts, so the upper half is stored during block NBLK/2 and the rows
    // up to the last block during the last block
    load_x<NB, false>(x, xc, 0, GH, lane);
    UPROF_MARK(8);
    block(0, R0{}, RN{}, XSched<NB, XS_GE_LOAD>{xc, lane});
    for (int s = 1; s < NBLK / 2; ++s) block(s, R0{}, RN{}, NoPf());
    block(NBLK / 2, RH{}, RN{}, XSched<NB, XS_GE_STORE>{xc, lane});
    if constexpr (NBLK / 2 < NBLK - 1) {
      for (int s = NBLK / 2 + 1; s < NBLK - 1; ++s) block(s, RH{}, RN{}, NoPf());
      block(NBLK - 1, RH{}, RN{}, XSched<NB, XS_GE_STORE2>{xc, lane});
      store_x<NB>(x, xc, NB / 8 - 4, NB / 8, lane);
    } else {
      store_x<NB>(x, xc, GH, NB / 8, lane);
    }
  } else {
    load_x<NB>(x, xc, 0, NB / 8, lane);
    UPROF_MARK(8);
    for (int s = 0; s < NBLK; ++s) block(s, R0{}, RN{}, NoPf());
    store_x<NB>(x, xc, 0, NB / 8, lane);
  }
  UPROF_MARK(6);
}

#ifdef TQR_PROF_L2
__device__ unsigned long long g_l2prof[8];
#define L2P_DECL long long _l2t = clock64()
#define L2P_MARK(k)                                                         \
  do {                                                                      \
    if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == 224)) {     \
      const long long _n = clock64();                                       \
      atomicAdd(&g_l2prof[(k) + (threadIdx.x ? 4 : 0)], (unsigned long long)(_n - _l2t)); \
      _l2t = _n;                                                            \
    }                                                                       \
  } while (0)
#else
#define L2P_DECL
#define L2P_MARK(k) \
  do {              \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// panel item: Householder QR of one tile (GE), of [R_piv; R_i] (TT) or of
// [R_piv; A_i] (TS), ib = 32 columns at a time, each block in four groups of
// 8 columns.  Within a group: one panel row (or two) per thread in
// registers, per column one 8-value warp reduce-scatter gives the norm and
// the dots with the group's later columns (dlarfg + reflector application,
// two CTA barriers per column).  After a group: one DMMA pass
// V_g^T [V_g | A_rest] (K = rows split over warps) yields the group Gram
// (-> T_g) and W; A_rest -= V_g T_g^T W on DMMA.  After the block: the
// 32x32 Gram V^T V on DMMA, T_b by back substitution, and the block
// reflector applied to the trailing columns of the tile(s) on DMMA.
//
// Stacked panel rows (P, panel-local): GE rows = tile rows rb0..NB-1 (the
// diagonal row of column j is row j); TT/TS rows 0..IB-1 = pivot block rows
// rb0.. (diagonal row j = row j), rows IB.. = bottom tile rows 0.. .

__device__ __forceinline__ unsigned long long ptimer() {
  unsigned long long tt;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tt));
  return tt;
}

// Global -> shared copy of `total` elements, element e read by ld(e) and
// written by st(e, v): eight loads per thread are in flight before their
// stores (a plain loop serializes one global-memory latency per element).
template <class LD, class ST>
__device__ __forceinline__ void batched_copy(int total, int tid, LD ld, ST st) {
  for (int e0 = tid; e0 < total; e0 += 8 * NT) {
    double v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int e = e0 + t * NT;
      v[t] = e < total ? ld(e) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int e = e0 + t * NT;
      if (e < total) st(e, v[t]);
    }
  }
}

template <int NB, int MODE>
__device__ __forceinline__ double vmask_p(double v, int row, int col) {
  // reflector entry of P row `row`, block column `col`
  if (MODE == GE) return row > col ? v : (row == col ? 1.0 : 0.0);
  return row >= IB ? v : (row == col ? 1.0 : 0.0);
}

// C(8 x 8*NBK) += V(:, cv0..cv0+7)^T * [V(:, cv0..cv0+7) | P(:, cv0+8..)]
// over rows [k0, k1) (multiple of 4), one warp; n-block 0 is the group's
// own reflectors (masked, -> Gram), the rest raw panel columns.  Lane (r,c)
// holds C[r][8nb + 2c + i].
template <int NB, int MODE, int NBK>
__device__ __forceinline__ void tn_acc(double (&acc)[NBK][2], const double* P, int cv0, int k0, int k1, int lane) {
  constexpr int PLD = NB + IB + 4;
  const int r = lane >> 2, c = lane & 3;
  for (int k = k0; k < k1; k += 4) {
    const int row = k + c;
    const double a = vmask_p<NB, MODE>(P[row + (cv0 + r) * PLD], row, cv0 + r);
    dmma(acc[0], a, a);  // B(k=c, n=r) = V[row][cv0+r]: the same element as this lane's A
#pragma unroll
    for (int nb = 1; nb < NBK; ++nb) dmma(acc[nb], a, P[row + (cv0 + 8 * nb + r) * PLD]);
  }
}

// Trailing update of the columns right of panel block b (8 columns per warp,
// register-resident) — a separate non-inlined function so that its register
// allocation does not compete with the panel's live state.
// The chunks holding the next panel block's columns (ch < IB/8) are
// forwarded into the stacked panel P in shared memory (P is dead during the
// trailing update) instead of being stored and reloaded: GE keeps only the
// block's final R rows (< rb0 + IB) for global memory, TT/TS forward every
// row they hold (the next block's write-back stores them).
template <int NB, int MODE>
__device__ __noinline__ void panel_trailing(double* at, double* rt, const double* Vs, const double* Ts, int b, int warp,
                                            int lane, double* P, int ch_begin = -1, int ch_end = 1 << 30,
                                            int ch_step = NW) {
  constexpr int PLD = Smem<NB>::PLD;
  const int rb0 = b * IB;
  const int nch = (NB - rb0 - IB) / 8;
  const int g0 = (MODE == GE) ? rb0 / 8 : 0;
  const int g1 = (MODE == TT) ? (rb0 + IB) / 8 : NB / 8;
  constexpr int GH = NB / 16;  // row groups of the upper half
  // the rows of the lower half load while the first GEMM runs on the upper
  // half (own scoreboard: see update_consume) when the block spans both
  const bool split = g0 < GH && g1 > GH;
  // (default: chunk ch on warp ch mod NW; the look-ahead panel gives each
  // warp group its own chunk range)
  for (int ch = ch_begin < 0 ? warp : ch_begin; ch < min(nch, ch_end); ch += ch_step) {
    const int col = rb0 + IB + ch * 8;
    double* const xc = at + size_t(col) * NB;
    double x[NB / 8][2];
    double* top = (MODE == GE) ? nullptr : rt + size_t(col) * NB + rb0;
    if (split) {
      load_x<NB>(x, xc, g0, GH, lane);
      auto lower = [&](auto&) { load_x<NB, false>(x, xc, GH, g1, lane); };
      warp_apply<NB, true, (MODE == TS ? 2 : MODE), 0, NB / IB, NoPf, decltype(lower)>(
          x, g0 / (IB / 8), g1 / (IB / 8), Vs, Ts, top, lane, nullptr, b, NoPf(), lower);
    } else {
      load_x<NB>(x, xc, g0, g1, lane);
      warp_apply<NB, true, (MODE == TS ? 2 : MODE)>(x, g0 / (IB / 8), g1 / (IB / 8), Vs, Ts, top, lane, nullptr, b);
    }
#ifndef TQR_NO_PANEL_FWD
    if (ch < IB / 8) {
      const int pc = ch * 8 + (lane >> 2), c2 = 2 * (lane & 3);
      const int gs = (MODE == GE) ? (rb0 + IB) / 8 : g0;  // first forwarded row group
      const int poff = (MODE == GE) ? -(rb0 + IB) : IB;    // P row of a tile row
      if (MODE == GE) store_x<NB>(x, xc, g0, gs, lane);
#pragma unroll
      for (int g = 0; g < NB / 8; ++g)
        if (g >= gs && g < g1)
          *reinterpret_cast<double2*>(P + poff + 8 * g + c2 + pc * PLD) = make_double2(x[g][0], x[g][1]);
      continue;
    }
#endif
    store_x<NB>(x, xc, g0, g1, lane);
  }
}

template <int NB, int MODE>
__device__ void panel_item(double* sm, double* at /*GE: tile; TT/TS: bottom tile (i,k)*/,
                           double* rt /*TT/TS: pivot tile (piv,k)*/, double* tslot, int tid,
                           unsigned long long* prof = nullptr) {
  using S = Smem<NB>;
  constexpr int PLD = S::PLD, LDW = S::LDW;
  const int warp = tid >> 5, lane = tid & 31;
  double* P = sm + S::P_P;
  double* Vs = sm + S::P_V;
  double* Ts = sm + S::P_T;
  double* G = sm + S::P_G;    // G[l + j*IB] = v_l . v_j
  double* Tp = sm + S::P_TT;  // T_b plain, row-major Tp[i*IB + j]
  double* WP = sm + S::P_WP;  // [warp][8][LDW] partial W
  double* W = sm + S::P_W;    // [8][LDW]
  double* Tg = sm + S::P_TG;  // 8x8 group T, Tg[i + j*8]
  double* part = sm + S::P_PART;
  double* drow = sm + S::P_DROW;
  double* sbuf = sm + S::P_SBUF;
  double* tau_s = sm + S::P_SC;
  double* taut_s = tau_s + IB;  // tau = 2 / v^T v of the stored v (T's diagonal)
  double* beta_s = tau_s + 2 * IB;
  const int t = tid;
  unsigned long long tp = (prof && tid == 0) ? ptimer() : 0;
  auto mark = [&](int ph) {
    if (prof && tid == 0) {
      const unsigned long long t2 = ptimer();
      atomicAdd(prof + MODE * 16 + ph, t2 - tp);
      tp = t2;
    }
  };

  for (int b = 0; b < NB / IB; ++b) {
    const int rb0 = b * IB;
    const int nrows = (MODE == GE) ? NB - rb0 : (MODE == TT ? IB + rb0 + IB : IB + NB);
    // ---- load the stacked panel into smem
#ifndef TQR_NO_PANEL_FWD
    const bool fwd = b > 0;  // rows forwarded into P by the previous block's trailing update
#else
    const bool fwd = false;
#endif
    // (every shape below has a compile-time row count: GE loads only block
    // 0, TT's bottom part is always IB rows, TS's is NB rows at block 0)
    if (MODE == GE) {
      if (!fwd)
        batched_copy(
            NB * IB, tid, [&](int e) { return __ldcg(at + e % NB + size_t(e / NB) * NB); },
            [&](int e, double v) { P[e % NB + (e / NB) * PLD] = v; });
    } else {
      // pivot triangle and the bottom rows not forwarded by the previous
      // block (TT: rows rb0 .. rb0+IB-1; TS: all NB rows, block 0 only)
      constexpr int NBR = (MODE == TT) ? IB : NB;
      const int rf = (MODE == TT) ? rb0 : 0;
      const int tot = IB * IB + ((MODE == TT || !fwd) ? NBR * IB : 0);
      batched_copy(
          tot, tid,
          [&](int e) {
            if (e < IB * IB) {
              const int r = e % IB, c = e / IB;
              return (r <= c) ? __ldcg(rt + (rb0 + r) + size_t(rb0 + c) * NB) : 0.0;
            }
            const int f = e - IB * IB, rr = rf + f % NBR, c = f / NBR;
            return (MODE == TS || rr <= rb0 + c) ? __ldcg(at + rr + size_t(rb0 + c) * NB) : 0.0;
          },
          [&](int e, double v) {
            if (e < IB * IB) {
              P[e % IB + (e / IB) * PLD] = v;
            } else {
              const int f = e - IB * IB;
              P[IB + rf + f % NBR + (f / NBR) * PLD] = v;
            }
          });
    }
    csync();
    mark(0);
    // rows owned by this thread: t and t+NT
    const int r0w = t, r1w = t + NT;
    const bool own0 = r0w < nrows, own1 = MODE != GE && r1w < nrows;  // GE: nrows <= NT
    auto in_vec = [&](int r, int j) {  // P row r belongs to reflector j's vector part
      if (MODE == GE) return r > j;
      if (MODE == TT) return r >= IB && r <= IB + rb0 + j;
      return r >= IB;
    };
    for (int gq = 0; gq < IB / 8; ++gq) {
      const int c0 = 8 * gq;
      // ---- level-2 on columns c0..c0+7 (registers: 8 values per owned row)
      double rv0[8], rv1[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        rv0[c] = own0 ? P[r0w + (c0 + c) * PLD] : 0.0;
        rv1[c] = own1 ? P[r1w + (c0 + c) * PLD] : 0.0;
      }
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        L2P_DECL;
        const int j = c0 + jj;
        double* partj = part + (jj & 1) * (NW * 8);  // double-buffered by column parity
        double* drowj = drow + (jj & 1) * 8;
        if (t == j) {
#pragma unroll
          for (int c = 0; c < 8; ++c) drowj[c] = rv0[c];
        }
        const bool iv0 = own0 && in_vec(r0w, j), iv1 = own1 && in_vec(r1w, j);
        double x0 = iv0 ? rv0[jj] : 0.0, x1 = iv1 ? rv1[jj] : 0.0;
        // products of x with the group's 8 columns, reduce-scattered over the
        // warp (lane L ends with value v(L) = 4*bit4 + 2*bit3 + bit2 summed
        // over its 32 lanes) into partj[warp][v]
        auto reduce8 = [&](double xa, double xb) {
          double d[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) d[c] = (MODE == GE) ? xa * rv0[c] : fma(xb, rv1[c], xa * rv0[c]);
          const bool u4 = lane & 16;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double snd = u4 ? d[i] : d[i + 4], kp = u4 ? d[i + 4] : d[i];
            d[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
          }
          const bool u3 = lane & 8;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const double snd = u3 ? d[i] : d[i + 2], kp = u3 ? d[i + 2] : d[i];
            d[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
          }
          const bool u2 = lane & 4;
          {
            const double snd = u2 ? d[0] : d[1], kp = u2 ? d[1] : d[0];
            d[0] = kp + __shfl_xor_sync(0xffffffffu, snd, 4);
          }
          d[0] += __shfl_xor_sync(0xffffffffu, d[0], 2);
          d[0] += __shfl_xor_sync(0xffffffffu, d[0], 1);
          if ((lane & 3) == 0) partj[warp * 8 + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1)] = d[0];
        };
        // every warp: lane v (mod 8) sums value v over the warps (the same
        // tree in every warp, so every warp holds bitwise the same values)
        const int v = lane & 7;
        auto sum8 = [&]() {
          double pw[NW];
#pragma unroll
          for (int w = 0; w < NW; ++w) pw[w] = partj[w * 8 + v];
#pragma unroll
          for (int h = NW / 2; h >= 1; h >>= 1)
#pragma unroll
            for (int w = 0; w < h; ++w) pw[w] += pw[w + h];
          return pw[0];
        };
        // dlarfg scalars (redundantly in every warp, no second barrier).
        // Common path: alpha^2 + ||x||^2 and every product in range.  Rare
        // path (CTA-uniform: every warp holds the same sums) — dnrm2-style
        // scaling: ||x|| tiny/zero or huge, or a product overflowed: the
        // column's max |x| (one more reduction) gives a power-of-two scale
        // 2^-ex; the products are redone with x' = 2^-ex x (||x'|| ~ 1,
        // |x' a| <= |a|, the norm term x' x'), and the scalars follow
        // dlarfg on the exact scales.
        reduce8(x0, x1);
        L2P_MARK(0);
        csync();
        L2P_MARK(1);
        const double alpha = drowj[jj];  // row j (written before the barrier)
        double D = sum8();
        const double xn2 = __shfl_sync(0xffffffffu, D, jj);
        // the range check is issued first and resolves beside the scalars'
        // dependency chain
        const bool rare = __any_sync(0xffffffffu, !(xn2 >= 0x1p-900 && fma(alpha, alpha, xn2) <= 0x1p900) ||
                                                      !isfinite(D));
        // scal_d: 1/(alpha - beta) in the common path; in the scaled path it
        // multiplies both the products D' (w_c = a_jc + scal D_c) and x'
        double tau, scal_d, beta;
        dlarfg_scalars(alpha, xn2, tau, scal_d, beta);
        if (__builtin_expect(rare, 0)) {
          double m = fmax(iv0 ? fabs(x0) : 0.0, iv1 ? fabs(x1) : 0.0);
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
          if (lane == 0) sbuf[warp] = m;
          csync();
          double amax = 0.0;
#pragma unroll
          for (int w = 0; w < NW; ++w) amax = fmax(amax, sbuf[w]);
          tau = scal_d = 0.0;
          beta = alpha;
          if (amax != 0.0) {  // (amax == 0: x = 0 below the diagonal, H = I)
            const int ex = ilogb(amax);
            const double xsc = ldexp(1.0, -ex);
            x0 *= xsc;  // from here on x' (the reflector is v = x' scal_d)
            x1 *= xsc;
            if (iv0) rv0[jj] = x0;  // the norm term of the products is x' x'
            if (iv1) rv1[jj] = x1;
            reduce8(x0, x1);
            csync();
            D = sum8();  // D'_c = 2^-ex D_c
            const double xn2s = __shfl_sync(0xffffffffu, D, jj);  // ||x'||^2 in [1, rows]
            if (fabs(alpha) >= ldexp(1.0, ex + 500)) {
              // ||x|| / |alpha| < 2^-490: dlapy2(alpha, xnorm) = |alpha| in
              // fp64, so beta = -alpha, tau = 2, scal = 1 / (2 alpha)
              tau = 2.0;
              beta = -alpha;
              scal_d = ldexp(0.5 / alpha, ex);
            } else {
              // dlarfg on the scaled column: beta = 2^ex beta', and with
              // scal = 2^-ex scal': scal D = scal' D', v = x scal = x' scal'
              dlarfg_scalars(ldexp(alpha, -ex), xn2s, tau, scal_d, beta);
              beta = ldexp(beta, ex);
            }
          }
        }
        L2P_MARK(2);
        const double sv = tau * (drowj[v] + scal_d * D);
        if (tid == 0) {
          tau_s[j] = tau;
          beta_s[j] = beta;
        }
        if (tau != 0.0) {
          double s[8];
#pragma unroll
          for (int c = jj + 1; c < 8; ++c) s[c] = __shfl_sync(0xffffffffu, sv, c);
          if (iv0) {
            const double xs = x0 * scal_d;
#pragma unroll
            for (int c = jj + 1; c < 8; ++c) rv0[c] -= s[c] * xs;
            rv0[jj] = xs;
          }
          if (iv1) {
            const double xs = x1 * scal_d;
#pragma unroll
            for (int c = jj + 1; c < 8; ++c) rv1[c] -= s[c] * xs;
            rv1[jj] = xs;
          }
          if (t == j) {
#pragma unroll
            for (int c = jj + 1; c < 8; ++c) rv0[c] -= s[c];
          }
        }
        if (t == j) rv0[jj] = beta;
        L2P_MARK(3);
        mark(7);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (own0) P[r0w + (c0 + c) * PLD] = rv0[c];
        if (own1) P[r1w + (c0 + c) * PLD] = rv1[c];
      }
      csync();
      mark(1);
      // ---- group update: W = V_g^T [V_g | A_rest] (DMMA, K = rows over warps)
      if (gq < IB / 8 - 1) {
        const int ncol = IB - c0 - 8;  // 24, 16, 8
        // rows that can hold nonzero reflector entries of this group
        const int klo = (MODE == GE) ? (c0 & ~3) : 0;
        const int khi = (MODE == GE) ? nrows : (MODE == TT ? IB + rb0 + c0 + 8 : nrows);
        const int ksteps = (khi - klo + 3) >> 2;
        const int per = (ksteps + NW - 1) / NW;
        const int ka = klo + 4 * per * warp, kb = min(khi, ka + 4 * per);
        double acc[4][2];
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) acc[nb][0] = acc[nb][1] = 0.0;
        if (ka < kb) {
          // rows beyond nrows are read as zero: clamp to a multiple of 4 within P
          const int kbb = ((kb - ka + 3) & ~3) + ka;
          if (ncol == 24)
            tn_acc<NB, MODE, 4>(acc, P, c0, ka, kbb, lane);
          else if (ncol == 16)
            tn_acc<NB, MODE, 3>(reinterpret_cast<double(&)[3][2]>(acc), P, c0, ka, kbb, lane);
          else
            tn_acc<NB, MODE, 2>(reinterpret_cast<double(&)[2][2]>(acc), P, c0, ka, kbb, lane);
        }
        {
          const int r = lane >> 2, c = lane & 3;
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) {
            WP[(warp * 8 + r) * LDW + 8 * nb + 2 * c] = acc[nb][0];
            WP[(warp * 8 + r) * LDW + 8 * nb + 2 * c + 1] = acc[nb][1];
          }
        }
        csync();
        // warps 1.. sum W_rest over the warps while warp 0 sums the group
        // Gram and computes T_g from it (one CTA barrier for both)
        if (warp > 0) {
          for (int e = tid - 32; e < 8 * ncol; e += NT - 32) {
            const int jr = e / ncol, cc = 8 + e % ncol;
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) s += WP[(w * 8 + jr) * LDW + cc];
            W[jr * LDW + cc] = s;
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int jr = (lane >> 3) + 4 * h, cc = lane & 7;
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) s += WP[(w * 8 + jr) * LDW + cc];
            W[jr * LDW + cc] = s;
          }
          __syncwarp();
        }
        // T_g (8x8) = (diag(1/tau) + striu(G_g))^-1 by back substitution;
        // lane cc owns column cc
        if (warp == 0 && lane < 8) {
          const int cc = lane;
          double col[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) col[i] = 0.0;
#pragma unroll
          for (int i = 7; i >= 0; --i) {
            double v = 0.0;
            if (i == cc) v = tau_s[c0 + i];
            if (i < cc) {
              double s = 0.0;
#pragma unroll
              for (int l = i + 1; l < 8; ++l)
                if (l <= cc) s += W[i * LDW + l] * col[l];
              v = -tau_s[c0 + i] * s;
            }
            col[i] = v;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) Tg[i + cc * 8] = col[i];
        }
        csync();
        // W_rest <- T_g^T W_rest
        for (int e = tid; e < 8 * ncol; e += NT) {
          const int jr = e / ncol, cc = 8 + e % ncol;
          double s = 0.0;
#pragma unroll
          for (int l = 0; l < 8; ++l)
            if (l <= jr) s += Tg[l + jr * 8] * W[l * LDW + cc];
          WP[jr * LDW + cc] = s;  // reuse warp-0 slab of WP as the result
        }
        csync();
        // A_rest -= V_g W_rest: m-blocks of 8 rows round-robin over warps
        {
          const int r = lane >> 2, c = lane & 3;
          const int mlo = klo >> 3, mhi = (khi + 7) >> 3;
          for (int mb = mlo + warp; mb < mhi; mb += NW) {
            const int row = 8 * mb + r;
            // A fragments: V[row][c0 + 4kk + c], k = reflector index
            double a0 = vmask_p<NB, MODE>(P[row + (c0 + c) * PLD], row, c0 + c);
            double a1 = vmask_p<NB, MODE>(P[row + (c0 + 4 + c) * PLD], row, c0 + 4 + c);
            for (int nb = 0; nb < ncol / 8; ++nb) {
              const int cb = c0 + 8 + 8 * nb;
              double acc2[2] = {0.0, 0.0};
              const double b0 = WP[c * LDW + 8 + 8 * nb + r];
              const double b1 = WP[(4 + c) * LDW + 8 + 8 * nb + r];
              dmma(acc2, a0, b0);
              dmma(acc2, a1, b1);
              if (row < nrows) {
                P[8 * mb + r + (cb + 2 * c) * PLD] -= acc2[0];
                P[8 * mb + r + (cb + 2 * c + 1) * PLD] -= acc2[1];
              }
            }
          }
        }
        csync();
        mark(2);
      }
    }
    // ---- block Gram G = V^T V (the 10 upper 8x8 blocks of 32x32) on DMMA.
    // T's consistency with the stored V sets the orthogonality of the block
    // reflector (I - V T V^T is orthogonal iff T^-1 + T^-T = V^T V), so G is
    // accumulated compensated: every 8 rows are formed from zero (two chained
    // DMMAs) and added error-free (TwoSum) into a hi/lo pair.  The row range
    // holding the block pair's nonzeros is split in two halves: 20 units on
    // the 8 warps; the halves' hi/lo are summed in double-double and rounded
    // once in the combine pass below.
    {
      double* Glo = Tp;  // half 0 low parts (Tp is first written after the combine)
      double* G1 = WP;   // half 1: [pair][hi 64 | lo 64]
      const int r = lane >> 2, c = lane & 3;
      for (int u = warp; u < 20; u += NW) {
        const int pr = u >> 1, half = u & 1;
        const int mb = pr < 4 ? 0 : (pr < 7 ? 1 : (pr < 9 ? 2 : 3));
        const int nbb = pr < 4 ? pr : (pr < 7 ? pr - 3 : (pr < 9 ? pr - 5 : 3));
        // GE: V's columns 8nbb.. are zero above P row 8nbb; TT: column block mb
        // (the shorter, mb <= nbb) ends at bottom row rb0 + 8mb + 7
        const int klo = (MODE == GE) ? 8 * nbb : 0;
        const int khi = (MODE == TT) ? IB + rb0 + 8 * mb + 8 : (nrows + 3) & ~3;
        const int mid = klo + (((khi - klo) >> 1) & ~7);
        const int k0 = half ? mid : klo, k1 = half ? khi : mid;
        double hi[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, lo[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        for (int k = k0; k < k1; k += 16) {
          double t[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int row = k + 4 * h + c;
            if (k + 4 * h < k1) {
              const double a = vmask_p<NB, MODE>(P[row + (8 * mb + r) * PLD], row, 8 * mb + r);
              const double bv = vmask_p<NB, MODE>(P[row + (8 * nbb + r) * PLD], row, 8 * nbb + r);
#ifdef TQR_GRAM_PLAIN
              dmma(hi[h >> 1], a, bv);
#else
              dmma(t[h >> 1], a, bv);
#endif
            }
          }
#ifndef TQR_GRAM_PLAIN
#pragma unroll
          for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              double s2, er;
              two_sum(s2, er, hi[q][e], t[q][e]);
              hi[q][e] = s2;
              lo[q][e] += er;
            }
#endif
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double s2, er;
          two_sum(s2, er, hi[0][e], hi[1][e]);
          const double l2 = er + (lo[0][e] + lo[1][e]);
          const int idx = (8 * mb + r) + (8 * nbb + 2 * c + e) * IB;
          if (half == 0) {
            G[idx] = s2;
            Glo[idx] = l2;
          } else {
            G1[pr * 128 + 2 * lane + e] = s2;
            G1[pr * 128 + 64 + 2 * lane + e] = l2;
          }
        }
      }
      csync();
      // combine the halves (double-double), round once; tau of each reflector
      // from its stored v (see the T step)
      for (int e = tid; e < 640; e += NT) {
        const int pr = e >> 6, w = e & 63, ln = w >> 1;
        const int mb = pr < 4 ? 0 : (pr < 7 ? 1 : (pr < 9 ? 2 : 3));
        const int nbb = pr < 4 ? pr : (pr < 7 ? pr - 3 : (pr < 9 ? pr - 5 : 3));
        const int i = 8 * mb + (ln >> 2), j = 8 * nbb + 2 * (ln & 3) + (w & 1);
        const int idx = i + j * IB;
        double s2, er;
        two_sum(s2, er, G[idx], G1[pr * 128 + w]);
        const double gv = s2 + (er + (Glo[idx] + G1[pr * 128 + 64 + w]));
        G[idx] = gv;
        if (i == j) taut_s[i] = tau_s[i] != 0.0 ? 2.0 / gv : 0.0;
      }
    }
    csync();
    mark(5);
    // ---- T_b = U^-1, U = diag(G)/2 + striu(G): dlarft (forward, columnwise)
    // with each reflector's tau taken as 2 / (v^T v) of its stored v instead
    // of dlarfg's (beta - alpha) / beta (equal in exact arithmetic; this one
    // makes every H_j = I - tau v v^T orthogonal to ~1 ulp); tau = 0
    // (x = 0, H_j = I) is kept:
    // the four 8x8 diagonal blocks by back substitution (lane = column),
    // then two block levels T12 = -T11 G12 T22 with all threads
    // (warps 4..7 zero the six strictly-lower 8x8 blocks meanwhile; every
    // upper block is written by the levels below)
    if (warp >= 4) {
      for (int e = tid - 128; e < 6 * 64; e += NT - 128) {
        const int k = e >> 6, bi = k < 1 ? 1 : (k < 3 ? 2 : 3), bj = k < 1 ? 0 : (k < 3 ? k - 1 : k - 3);
        Tp[(bi * 8 + ((e & 63) >> 3)) * IB + bj * 8 + (e & 7)] = 0.0;
      }
    }
    if (warp < 4 && lane < 8) {
      const int g0 = warp * 8, cc = lane;
      double col[8], tv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#ifdef TQR_TAU_DLARFG
        tv[i] = tau_s[g0 + i];
#else
        tv[i] = taut_s[g0 + i];
#endif
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        double v = 0.0;
        if (i == cc) v = tv[i];
        if (i < cc) {
          double s = 0.0;
#pragma unroll
          for (int l = i + 1; l < 8; ++l)
            if (l <= cc) s += G[(g0 + i) + (g0 + l) * IB] * col[l];
          v = -tv[i] * s;
        }
        col[i] = v;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) Tp[(g0 + i) * IB + g0 + cc] = col[i];
    }
    csync();
    double* M = WP;  // scratch, row-major IB x IB
    // level 1: blocks (0,1) and (2,3): M = G12 T22, then T12 = -T11 M
    if (tid < 128) {
      const int pb = tid >> 6, e = tid & 63, i = e >> 3, jx = e & 7;
      const int a0 = 16 * pb, b0 = a0 + 8;
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < 8; ++l) s += G[(a0 + i) + (b0 + l) * IB] * Tp[(b0 + l) * IB + b0 + jx];
      M[(a0 + i) * IB + b0 + jx] = s;
    }
    csync();
    if (tid < 128) {
      const int pb = tid >> 6, e = tid & 63, i = e >> 3, jx = e & 7;
      const int a0 = 16 * pb, b0 = a0 + 8;
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < 8; ++l) s += Tp[(a0 + i) * IB + a0 + l] * M[(a0 + l) * IB + b0 + jx];
      Tp[(a0 + i) * IB + b0 + jx] = -s;
    }
    csync();
    // level 2: rows 0..15 x cols 16..31
    {
      const int i = tid >> 4, jx = tid & 15;
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < 16; ++l) s += G[i + (16 + l) * IB] * Tp[(16 + l) * IB + 16 + jx];
      M[i * IB + 16 + jx] = s;
    }
    csync();
    {
      const int i = tid >> 4, jx = tid & 15;
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < 16; ++l) s += Tp[i * IB + l] * M[l * IB + 16 + jx];
      Tp[i * IB + 16 + jx] = -s;
    }
    csync();
    mark(6);
    // ---- write the block back to HBM, stage V and T for the trailing update
    for (int e = tid; e < IB * IB; e += NT) {
      const int i = e % IB, j = e / IB;
      const double v = Tp[i * IB + j];
      Ts[swz(i, j)] = v;
      tslot[i + size_t(rb0 + j) * IB] = v;
    }
    csync();  // Vs overwrites Tp / G / the scalars
    // (warp per column, lane per row: row counts are multiples of 32, so
    // no integer division per element)
    if (MODE == GE) {
      for (int c = warp; c < IB; c += NW)
        for (int r = lane; r < nrows; r += 32) {
          const double v = P[r + c * PLD];
          at[(rb0 + r) + size_t(rb0 + c) * NB] = v;
          Vs[swz(rb0 + r, c)] = (r > c) ? v : (r == c ? 1.0 : 0.0);
        }
    } else {
      const int nb_rows = nrows - IB;
      for (int c = warp; c < IB; c += NW) {
        if (lane <= c) rt[(rb0 + lane) + size_t(rb0 + c) * NB] = P[lane + c * PLD];
        for (int rr = lane; rr < nb_rows; rr += 32) {
          const bool live = (MODE == TS) || (rr <= rb0 + c);
          const double v = live ? P[IB + rr + c * PLD] : 0.0;
          if (live) at[rr + size_t(rb0 + c) * NB] = v;
          Vs[swz(rr, c)] = v;
        }
      }
    }
    csync();
    mark(3);
    // ---- trailing update of columns rb0+IB .. NB on DMMA, 8 columns per warp
    panel_trailing<NB, MODE>(at, rt, Vs, Ts, b, warp, lane, P);
    csync();
    mark(4);
  }
}

// ---------------------------------------------------------------------------
// Look-ahead panel item: the same factorization as panel_item, with the
// compute warps split in two groups once block 0 is factored.  Warps 0..3
// (FG) apply block b-1's reflectors to the 32 columns of block b (forwarded
// into the stacked panel), then run block b's level-2 sweep and group
// updates (128 threads, up to three panel rows per thread) while warps 4..7
// (UG) apply block b-1 to the columns right of block b.  Both groups meet
// for the block Gram, T_b, the write-back and the staging of V_b (all eight
// warps, as in panel_item).  The level-2 chain is latency-bound and leaves the
// DMMA pipe idle, the trailing update is DMMA-bound: they overlap instead of
// adding up.
template <int NB, int MODE>
__device__ void panel_item_la(double* sm, double* at /*GE: tile; TT/TS: bottom tile (i,k)*/,
                              double* rt /*TT/TS: pivot tile (piv,k)*/, double* tslot, int tid,
                              unsigned long long* prof = nullptr) {
  using S = Smem<NB>;
  constexpr int PLD = S::PLD, LDW = S::LDW, FW = S::FW, FT = FW * 32;
  const int warp = tid >> 5, lane = tid & 31;
  double* P = sm + S::P_P;
  double* Ts = sm + S::P_T;
  double* W = sm + S::L_W;    // [8][LDW]
  double* Tg = sm + S::L_TG;  // 8x8 group T, Tg[i + j*8]
  double* part = sm + S::L_PART;
  double* drow = sm + S::L_DROW;
  double* sbuf = sm + S::L_SBUF;
  double* tau_s = sm + S::L_SC;
  double* taut_s = tau_s + IB;
  double* beta_s = tau_s + 2 * IB;
  double* WP = sm + S::L_WP;  // [FW][8][LDW] partial W; T scratch
  double* Vs = sm + S::L_V;
  double* G = sm + S::L_G;    // G[l + j*IB] = v_l . v_j   (aliases Vs)
  double* Tp = sm + S::L_TT;  // T_b plain, row-major      (aliases Vs)
  double* G1 = sm + S::L_G1;  // Gram units' second halves (aliases Vs)
  double* Glo = Tp;           // first halves' low parts (Tp is first written after the combine)
  // One unit of the compensated block Gram (see panel_item): half `half` of
  // the row range of the 8x8 block pair pr.  Pairs of column groups 0..2 only
  // need those groups' reflectors, which are final once group 2's level-2
  // sweep is done: UG computes them while FG finishes the block.
  auto gram_unit = [&](int pr, int half, int rb0, int nrows) {
    const int r = lane >> 2, c = lane & 3;
    const int mb = pr < 4 ? 0 : (pr < 7 ? 1 : (pr < 9 ? 2 : 3));
    const int nbb = pr < 4 ? pr : (pr < 7 ? pr - 3 : (pr < 9 ? pr - 5 : 3));
    const int klo = (MODE == GE) ? 8 * nbb : 0;
    const int khi = (MODE == TT) ? IB + rb0 + 8 * mb + 8 : (nrows + 3) & ~3;
    const int mid = klo + (((khi - klo) >> 1) & ~7);
    const int k0 = half ? mid : klo, k1 = half ? khi : mid;
    double hi[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, lo[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int k = k0; k < k1; k += 16) {
      double tt[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int row = k + 4 * h + c;
        if (k + 4 * h < k1) {
          const double a = vmask_p<NB, MODE>(P[row + (8 * mb + r) * PLD], row, 8 * mb + r);
          const double bv = vmask_p<NB, MODE>(P[row + (8 * nbb + r) * PLD], row, 8 * nbb + r);
          dmma(tt[h >> 1], a, bv);
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double s2, er;
          two_sum(s2, er, hi[q][e], tt[q][e]);
          hi[q][e] = s2;
          lo[q][e] += er;
        }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double s2, er;
      two_sum(s2, er, hi[0][e], hi[1][e]);
      const double l2 = er + (lo[0][e] + lo[1][e]);
      const int idx = (8 * mb + r) + (8 * nbb + 2 * c + e) * IB;
      if (half == 0) {
        G[idx] = s2;
        Glo[idx] = l2;
      } else {
        G1[pr * 128 + 2 * lane + e] = s2;
        G1[pr * 128 + 64 + 2 * lane + e] = l2;
      }
    }
  };
  const int t = tid;
  const bool fg = warp < FW;
  auto fsync = [&]() { asm volatile("bar.sync 3, %0;\n" ::"n"(FT) : "memory"); };
  unsigned long long tp = (prof && tid == 0) ? ptimer() : 0;
  auto mark = [&](int ph) {
    if (prof && tid == 0) {
      const unsigned long long t2 = ptimer();
      atomicAdd(prof + MODE * 16 + ph, t2 - tp);
      tp = t2;
    }
  };

  for (int b = 0; b < NB / IB; ++b) {
    const int rb0 = b * IB;
    const int nrows = (MODE == GE) ? NB - rb0 : (MODE == TT ? IB + rb0 + IB : IB + NB);
    // the part of the stacked panel that is not forwarded by the trailing
    // update (see panel_item); it does not depend on block b-1 (GE loads
    // block 0 only; the pivot triangle and TT's new bottom rows are not
    // touched by earlier blocks), so for b > 0 UG loads it before its
    // trailing chunks.  lt: thread index within the loading group
    auto load_rest = [&](int lt) {
      const bool fwd = b > 0;
      if (MODE == GE) {
        if (!fwd) {
          for (int e0 = lt; e0 < NB * IB; e0 += 8 * FT) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int e = e0 + u * FT;
              v[u] = e < NB * IB ? __ldcg(at + e % NB + size_t(e / NB) * NB) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int e = e0 + u * FT;
              if (e < NB * IB) P[e % NB + (e / NB) * PLD] = v[u];
            }
          }
        }
      } else {
        constexpr int NBR = (MODE == TT) ? IB : NB;
        const int rf = (MODE == TT) ? rb0 : 0;
        const int tot = IB * IB + ((MODE == TT || !fwd) ? NBR * IB : 0);
        for (int e0 = lt; e0 < tot; e0 += 8 * FT) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * FT;
            double x = 0.0;
            if (e < tot) {
              if (e < IB * IB) {
                const int r = e % IB, c = e / IB;
                if (r <= c) x = __ldcg(rt + (rb0 + r) + size_t(rb0 + c) * NB);
              } else {
                const int f = e - IB * IB, rr = rf + f % NBR, c = f / NBR;
                if (MODE == TS || rr <= rb0 + c) x = __ldcg(at + rr + size_t(rb0 + c) * NB);
              }
            }
            v[u] = x;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * FT;
            if (e < tot) {
              if (e < IB * IB) {
                P[e % IB + (e / IB) * PLD] = v[u];
              } else {
                const int f = e - IB * IB;
                P[IB + rf + f % NBR + (f / NBR) * PLD] = v[u];
              }
            }
          }
        }
      }
    };
    if (!fg) {
      // UG: the loads, then block b-1's reflectors on the columns right of block b
      if (b > 0) {
        if (MODE != GE) load_rest(tid - FT);
        asm volatile("bar.arrive 4, %0;\n" ::"n"(NT) : "memory");  // panel loaded
        panel_trailing<NB, MODE>(at, rt, Vs, Ts, b - 1, warp, lane, P, IB / 8 + warp - FW, 1 << 30, NW - FW);
      }
      // the Gram pairs of column groups 0..2 (V_{b-1} staged in Vs is dead:
      // FG's chunks ended before its level-2 sweep, UG's just now)
      asm volatile("bar.sync 5, %0;\n" ::"n"(NT) : "memory");  // groups 0..2 are final in P
      for (int u = warp - FW; u < 12; u += NW - FW) {
        const int e6 = u >> 1;
        gram_unit(e6 < 3 ? e6 : (e6 < 5 ? e6 + 1 : 7), u & 1, rb0, nrows);
      }
    } else {
      // FG: block b-1's reflectors on block b's columns (one 8-column chunk
      // per warp, forwarded into P)
      if (b > 0) {
        panel_trailing<NB, MODE>(at, rt, Vs, Ts, b - 1, warp, lane, P, warp, IB / 8, FW);
        asm volatile("bar.sync 4, %0;\n" ::"n"(NT) : "memory");  // FG's chunks and UG's loads are in P
      } else {
        load_rest(tid);
        fsync();
      }
      mark(4);

      // rows owned by this thread: t, t + FT, t + 2 FT
      const int r0w = t, r1w = t + FT, r2w = t + 2 * FT;
      const bool own0 = r0w < nrows, own1 = r1w < nrows, own2 = MODE != GE && r2w < nrows;  // GE: nrows <= 2 FT
      auto in_vec = [&](int r, int j) {  // P row r belongs to reflector j's vector part
        if (MODE == GE) return r > j;
        if (MODE == TT) return r >= IB && r <= IB + rb0 + j;
        return r >= IB;
      };
      for (int gq = 0; gq < IB / 8; ++gq) {
        const int c0 = 8 * gq;
        // ---- level-2 on columns c0..c0+7 (registers: 8 values per owned row)
        double rv0[8], rv1[8], rv2[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          rv0[c] = own0 ? P[r0w + (c0 + c) * PLD] : 0.0;
          rv1[c] = own1 ? P[r1w + (c0 + c) * PLD] : 0.0;
          rv2[c] = own2 ? P[r2w + (c0 + c) * PLD] : 0.0;
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int j = c0 + jj;
          double* partj = part + (jj & 1) * (NW * 8);  // double-buffered by column parity
          double* drowj = drow + (jj & 1) * 8;
          if (t == j) {
#pragma unroll
            for (int c = 0; c < 8; ++c) drowj[c] = rv0[c];
          }
          const bool iv0 = own0 && in_vec(r0w, j), iv1 = own1 && in_vec(r1w, j), iv2 = own2 && in_vec(r2w, j);
          double x0 = iv0 ? rv0[jj] : 0.0, x1 = iv1 ? rv1[jj] : 0.0, x2 = iv2 ? rv2[jj] : 0.0;
          auto reduce8 = [&](double xa, double xb, double xc) {
            double d[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              d[c] = fma(xb, rv1[c], xa * rv0[c]);
              if (MODE != GE) d[c] = fma(xc, rv2[c], d[c]);
            }
            const bool u4 = lane & 16;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const double snd = u4 ? d[i] : d[i + 4], kp = u4 ? d[i + 4] : d[i];
              d[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
            }
            const bool u3 = lane & 8;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const double snd = u3 ? d[i] : d[i + 2], kp = u3 ? d[i + 2] : d[i];
              d[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
            }
            const bool u2 = lane & 4;
            {
              const double snd = u2 ? d[0] : d[1], kp = u2 ? d[1] : d[0];
              d[0] = kp + __shfl_xor_sync(0xffffffffu, snd, 4);
            }
            d[0] += __shfl_xor_sync(0xffffffffu, d[0], 2);
            d[0] += __shfl_xor_sync(0xffffffffu, d[0], 1);
            if ((lane & 3) == 0)
              partj[warp * 8 + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1)] = d[0];
          };
          const int v = lane & 7;
          auto sum8 = [&]() {
            double pw[FW];
#pragma unroll
            for (int w = 0; w < FW; ++w) pw[w] = partj[w * 8 + v];
#pragma unroll
            for (int h = FW / 2; h >= 1; h >>= 1)
#pragma unroll
              for (int w = 0; w < h; ++w) pw[w] += pw[w + h];
            return pw[0];
          };
          reduce8(x0, x1, x2);
          fsync();
          const double alpha = drowj[jj];  // row j (written before the barrier)
          double D = sum8();
          const double xn2 = __shfl_sync(0xffffffffu, D, jj);
          const bool rare = __any_sync(0xffffffffu, !(xn2 >= 0x1p-900 && fma(alpha, alpha, xn2) <= 0x1p900) ||
                                                        !isfinite(D));
          double tau, scal_d, beta;
          dlarfg_scalars(alpha, xn2, tau, scal_d, beta);
          if (__builtin_expect(rare, 0)) {  // scaled path, see panel_item
            double m = fmax(fmax(iv0 ? fabs(x0) : 0.0, iv1 ? fabs(x1) : 0.0), iv2 ? fabs(x2) : 0.0);
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) sbuf[warp] = m;
            fsync();
            double amax = 0.0;
#pragma unroll
            for (int w = 0; w < FW; ++w) amax = fmax(amax, sbuf[w]);
            tau = scal_d = 0.0;
            beta = alpha;
            if (amax != 0.0) {
              const int ex = ilogb(amax);
              const double xsc = ldexp(1.0, -ex);
              x0 *= xsc;
              x1 *= xsc;
              x2 *= xsc;
              if (iv0) rv0[jj] = x0;
              if (iv1) rv1[jj] = x1;
              if (iv2) rv2[jj] = x2;
              reduce8(x0, x1, x2);
              fsync();
              D = sum8();
              const double xn2s = __shfl_sync(0xffffffffu, D, jj);
              if (fabs(alpha) >= ldexp(1.0, ex + 500)) {
                tau = 2.0;
                beta = -alpha;
                scal_d = ldexp(0.5 / alpha, ex);
              } else {
                dlarfg_scalars(ldexp(alpha, -ex), xn2s, tau, scal_d, beta);
                beta = ldexp(beta, ex);
              }
            }
          }
          const double sv = tau * (drowj[v] + scal_d * D);
          if (tid == 0) {
            tau_s[j] = tau;
            beta_s[j] = beta;
          }
          if (tau != 0.0) {
            double sc[8];
#pragma unroll
            for (int c = jj + 1; c < 8; ++c) sc[c] = __shfl_sync(0xffffffffu, sv, c);
            if (iv0) {
              const double xs = x0 * scal_d;
#pragma unroll
              for (int c = jj + 1; c < 8; ++c) rv0[c] -= sc[c] * xs;
              rv0[jj] = xs;
            }
            if (iv1) {
              const double xs = x1 * scal_d;
#pragma unroll
              for (int c = jj + 1; c < 8; ++c) rv1[c] -= sc[c] * xs;
              rv1[jj] = xs;
            }
            if (iv2) {
              const double xs = x2 * scal_d;
#pragma unroll
              for (int c = jj + 1; c < 8; ++c) rv2[c] -= sc[c] * xs;
              rv2[jj] = xs;
            }
            if (t == j) {
#pragma unroll
              for (int c = jj + 1; c < 8; ++c) rv0[c] -= sc[c];
            }
          }
          if (t == j) rv0[jj] = beta;
          mark(7);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (own0) P[r0w + (c0 + c) * PLD] = rv0[c];
          if (own1) P[r1w + (c0 + c) * PLD] = rv1[c];
          if (own2) P[r2w + (c0 + c) * PLD] = rv2[c];
        }
        fsync();
        if (gq == 2) asm volatile("bar.arrive 5, %0;\n" ::"n"(NT) : "memory");  // groups 0..2 final: UG's Gram pairs
        mark(1);
        // ---- group update: W = V_g^T [V_g | A_rest] (DMMA, K = rows over the FW warps)
        if (gq < IB / 8 - 1) {
          const int ncol = IB - c0 - 8;  // 24, 16, 8
          const int klo = (MODE == GE) ? (c0 & ~3) : 0;
          const int khi = (MODE == GE) ? nrows : (MODE == TT ? IB + rb0 + c0 + 8 : nrows);
          const int ksteps = (khi - klo + 3) >> 2;
          const int per = (ksteps + FW - 1) / FW;
          const int ka = klo + 4 * per * warp, kb = min(khi, ka + 4 * per);
          double acc[4][2];
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) acc[nb][0] = acc[nb][1] = 0.0;
          if (ka < kb) {
            const int kbb = ((kb - ka + 3) & ~3) + ka;
            if (ncol == 24)
              tn_acc<NB, MODE, 4>(acc, P, c0, ka, kbb, lane);
            else if (ncol == 16)
              tn_acc<NB, MODE, 3>(reinterpret_cast<double(&)[3][2]>(acc), P, c0, ka, kbb, lane);
            else
              tn_acc<NB, MODE, 2>(reinterpret_cast<double(&)[2][2]>(acc), P, c0, ka, kbb, lane);
          }
          {
            const int r = lane >> 2, c = lane & 3;
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) {
              WP[(warp * 8 + r) * LDW + 8 * nb + 2 * c] = acc[nb][0];
              WP[(warp * 8 + r) * LDW + 8 * nb + 2 * c + 1] = acc[nb][1];
            }
          }
          fsync();
          if (warp > 0) {
            for (int e = tid - 32; e < 8 * ncol; e += FT - 32) {
              const int jr = e / ncol, cc = 8 + e % ncol;
              double sacc = 0.0;
#pragma unroll
              for (int w = 0; w < FW; ++w) sacc += WP[(w * 8 + jr) * LDW + cc];
              W[jr * LDW + cc] = sacc;
            }
          } else {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int jr = (lane >> 3) + 4 * h, cc = lane & 7;
              double sacc = 0.0;
#pragma unroll
              for (int w = 0; w < FW; ++w) sacc += WP[(w * 8 + jr) * LDW + cc];
              W[jr * LDW + cc] = sacc;
            }
            __syncwarp();
          }
          if (warp == 0 && lane < 8) {
            const int cc = lane;
            double col[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) col[i] = 0.0;
#pragma unroll
            for (int i = 7; i >= 0; --i) {
              double vv = 0.0;
              if (i == cc) vv = tau_s[c0 + i];
              if (i < cc) {
                double sacc = 0.0;
#pragma unroll
                for (int l = i + 1; l < 8; ++l)
                  if (l <= cc) sacc += W[i * LDW + l] * col[l];
                vv = -tau_s[c0 + i] * sacc;
              }
              col[i] = vv;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) Tg[i + cc * 8] = col[i];
          }
          fsync();
          for (int e = tid; e < 8 * ncol; e += FT) {
            const int jr = e / ncol, cc = 8 + e % ncol;
            double sacc = 0.0;
#pragma unroll
            for (int l = 0; l < 8; ++l)
              if (l <= jr) sacc += Tg[l + jr * 8] * W[l * LDW + cc];
            WP[jr * LDW + cc] = sacc;  // reuse warp-0 slab of WP as the result
          }
          fsync();
          {
            const int r = lane >> 2, c = lane & 3;
            const int mlo = klo >> 3, mhi = (khi + 7) >> 3;
            for (int mb = mlo + warp; mb < mhi; mb += FW) {
              const int row = 8 * mb + r;
              double a0 = vmask_p<NB, MODE>(P[row + (c0 + c) * PLD], row, c0 + c);
              double a1 = vmask_p<NB, MODE>(P[row + (c0 + 4 + c) * PLD], row, c0 + 4 + c);
              for (int nb = 0; nb < ncol / 8; ++nb) {
                const int cb = c0 + 8 + 8 * nb;
                double acc2[2] = {0.0, 0.0};
                const double b0 = WP[c * LDW + 8 + 8 * nb + r];
                const double b1 = WP[(4 + c) * LDW + 8 + 8 * nb + r];
                dmma(acc2, a0, b0);
                dmma(acc2, a1, b1);
                if (row < nrows) {
                  P[8 * mb + r + (cb + 2 * c) * PLD] -= acc2[0];
                  P[8 * mb + r + (cb + 2 * c + 1) * PLD] -= acc2[1];
                }
              }
            }
          }
          fsync();
          mark(2);
        }
      }
    }
    csync();  // block b is factored in P; block b-1 is applied to every column right of it
    // ---- block Gram (compensated), T_b, write-back, staging of V_b and T_b:
    // all eight warps, as in panel_item
    {
      // the pairs with column group 3 (two halves each: one unit per warp)
      {
        const int l4 = warp >> 1;
        gram_unit(l4 == 0 ? 3 : (l4 == 1 ? 6 : (l4 == 2 ? 8 : 9)), warp & 1, rb0, nrows);
      }
      csync();
      for (int e = tid; e < 640; e += NT) {
        const int pr = e >> 6, w = e & 63, ln = w >> 1;
        const int mb = pr < 4 ? 0 : (pr < 7 ? 1 : (pr < 9 ? 2 : 3));
        const int nbb = pr < 4 ? pr : (pr < 7 ? pr - 3 : (pr < 9 ? pr - 5 : 3));
        const int i = 8 * mb + (ln >> 2), j = 8 * nbb + 2 * (ln & 3) + (w & 1);
        const int idx = i + j * IB;
        double s2, er;
        two_sum(s2, er, G[idx], G1[pr * 128 + w]);
        const double gv = s2 + (er + (Glo[idx] + G1[pr * 128 + 64 + w]));
        G[idx] = gv;
        if (i == j) taut_s[i] = tau_s[i] != 0.0 ? 2.0 / gv : 0.0;
      }
    }
    csync();
    mark(5);
    // ---- T_b = U^-1 (dlarft with tau = 2 / v^T v), see panel_item
    if (warp >= 4) {
      for (int e = tid - 128; e < 6 * 64; e += NT - 128) {
        const int k = e >> 6, bi = k < 1 ? 1 : (k < 3 ? 2 : 3), bj = k < 1 ? 0 : (k < 3 ? k - 1 : k - 3);
        Tp[(bi * 8 + ((e & 63) >> 3)) * IB + bj * 8 + (e & 7)] = 0.0;
      }
    }
    if (warp < 4 && lane < 8) {
      const int g0 = warp * 8, cc = lane;
      double col[8], tv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) tv[i] = taut_s[g0 + i];
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        double vv = 0.0;
        if (i == cc) vv = tv[i];
        if (i < cc) {
          double sacc = 0.0;
#pragma unroll
          for (int l = i + 1; l < 8; ++l)
            if (l <= cc) sacc += G[(g0 + i) + (g0 + l) * IB] * col[l];
          vv = -tv[i] * sacc;
        }
        col[i] = vv;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) Tp[(g0 + i) * IB + g0 + cc] = col[i];
    }
    csync();
    double* M = WP;  // scratch, row-major IB x IB
    if (tid < 128) {
      const int pb = tid >> 6, e = tid & 63, i = e >> 3, jx = e & 7;
      const int a0 = 16 * pb, b0 = a0 + 8;
      double sacc = 0.0;
#pragma unroll
      for (int l = 0; l < 8; ++l) sacc += G[(a0 + i) + (b0 + l) * IB] * Tp[(b0 + l) * IB + b0 + jx];
      M[(a0 + i) * IB + b0 + jx] = sacc;
    }
    csync();
    if (tid < 128) {
      const int pb = tid >> 6, e = tid & 63, i = e >> 3, jx = e & 7;
      const int a0 = 16 * pb, b0 = a0 + 8;
      double sacc = 0.0;
#pragma unroll
      for (int l = 0; l < 8; ++l) sacc += Tp[(a0 + i) * IB + a0 + l] * M[(a0 + l) * IB + b0 + jx];
      Tp[(a0 + i) * IB + b0 + jx] = -sacc;
    }
    csync();
    {
      const int i = tid >> 4, jx = tid & 15;
      double sacc = 0.0;
#pragma unroll
      for (int l = 0; l < 16; ++l) sacc += G[i + (16 + l) * IB] * Tp[(16 + l) * IB + 16 + jx];
      M[i * IB + 16 + jx] = sacc;
    }
    csync();
    {
      const int i = tid >> 4, jx = tid & 15;
      double sacc = 0.0;
#pragma unroll
      for (int l = 0; l < 16; ++l) sacc += Tp[i * IB + l] * M[l * IB + 16 + jx];
      Tp[i * IB + 16 + jx] = -sacc;
    }
    csync();
    mark(6);
    // ---- write the block back to HBM, stage V and T for the trailing update
    for (int e = tid; e < IB * IB; e += NT) {
      const int i = e % IB, j = e / IB;
      const double vv = Tp[i * IB + j];
      Ts[swz(i, j)] = vv;
      tslot[i + size_t(rb0 + j) * IB] = vv;
    }
    csync();  // Vs overwrites Tp / G
    if (MODE == GE) {
      for (int c = warp; c < IB; c += NW)
        for (int r = lane; r < nrows; r += 32) {
          const double vv = P[r + c * PLD];
          at[(rb0 + r) + size_t(rb0 + c) * NB] = vv;
          Vs[swz(rb0 + r, c)] = (r > c) ? vv : (r == c ? 1.0 : 0.0);
        }
    } else {
      const int nb_rows = nrows - IB;
      for (int c = warp; c < IB; c += NW) {
        if (lane <= c) rt[(rb0 + lane) + size_t(rb0 + c) * NB] = P[lane + c * PLD];
        for (int rr = lane; rr < nb_rows; rr += 32) {
          const bool live = (MODE == TS) || (rr <= rb0 + c);
          const double vv = live ? P[IB + rr + c * PLD] : 0.0;
          if (live) at[rr + size_t(rb0 + c) * NB] = vv;
          Vs[swz(rr, c)] = vv;
        }
      }
    }
    csync();  // V_b, T_b staged: the groups split again
    mark(3);
  }
}

// The panel item the executor runs: the look-ahead form (TQR_PANEL_NO_LA:
// panel_item, one phase at a time on all eight warps).
template <int NB, int MODE>
__device__ __forceinline__ void panel_run(double* sm, double* at, double* rt, double* tslot, int tid,
                                          unsigned long long* prof = nullptr) {
#ifndef TQR_PANEL_NO_LA
  panel_item_la<NB, MODE>(sm, at, rt, tslot, tid, prof);
#else
  panel_item<NB, MODE>(sm, at, rt, tslot, tid, prof);
#endif
}

}  // namespace tqrk
