// Kernel tasks of the tiled QR (one CTA of 256 threads per work item):
//   update items  UNMQR / TTMQR / TSMQR on one 64-column slab   (qr.py:431-481)
//   panel items   GEQRT / TTQRT / TSQRT on one tile (pair)      (qr.py:421-471)
// Numerics follow LAPACK dgeqrt/dgemqrt/dtpqrt/dtpmqrt (compact WY with ib-
// blocked T), so V, R and T match the oracle's LAPACK replay.
#pragma once
#include "tqr_device.cuh"

namespace tqrk {

// Shared-memory carve-up (doubles).  Update items: Vs[2] + Ts[2].
// Panel items: P (stacked panel), Vs, Ts, G and per-column scalars.
template <int NB>
struct Smem {
  static constexpr int VS = NB * IB;  // one staged V block
  static constexpr int TS = IB * IB;
  static constexpr int PLD = NB + IB;  // panel leading dimension
  static constexpr int P = PLD * IB;
  // update layout
  static constexpr int U_V0 = 0, U_V1 = VS, U_T0 = 2 * VS, U_T1 = 2 * VS + TS, U_END = 2 * VS + 2 * TS;
  // panel layout
  static constexpr int P_P = 0, P_V = P, P_T = P + VS, P_G = P + VS + TS, P_SC = P + VS + 2 * TS;
  static constexpr int P_END = P_SC + 4 * IB + 8;
  static constexpr int END = U_END > P_END ? U_END : P_END;
  static constexpr size_t BYTES = size_t(END) * sizeof(double);
};

// ---------------------------------------------------------------------------
// update item: apply all ib-blocks of one factor's reflectors to a 64-column
// slab of the target tile(s), slab resident in registers for all blocks.

template <int NB, int MODE, bool TRANST>
__device__ void update_item(double* sm, const double* __restrict__ vt, const double* __restrict__ tt, double* xt,
                            double* topt, int slab, int tid) {
  using S = Smem<NB>;
  const int warp = tid >> 5, lane = tid & 31;
  const int col0 = slab * WS + warp * 8;
  double x[NB / 8][2];
  load_x<NB>(x, xt + size_t(col0) * NB, 0, NB / 8, lane);
  constexpr int NBLK = NB / IB;
  auto rows_of = [](int b, int& r0, int& r1) {
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
  };
  {
    const int b = TRANST ? 0 : NBLK - 1;
    int r0, r1;
    rows_of(b, r0, r1);
    stage_v<NB, MODE>(sm + S::U_V0, vt, b, r0, r1, tid);
    stage_t(sm + S::U_T0, tt, b, tid);
    cp_async_commit();
  }
  for (int s = 0; s < NBLK; ++s) {
    const int b = TRANST ? s : NBLK - 1 - s;
    if (s + 1 < NBLK) {
      const int bn = TRANST ? s + 1 : NBLK - 2 - s;
      int r0, r1;
      rows_of(bn, r0, r1);
      stage_v<NB, MODE>(sm + (((s + 1) & 1) ? S::U_V1 : S::U_V0), vt, bn, r0, r1, tid);
      stage_t(sm + (((s + 1) & 1) ? S::U_T1 : S::U_T0), tt, bn, tid);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    int r0, r1;
    rows_of(b, r0, r1);
    const double* Vs = sm + ((s & 1) ? S::U_V1 : S::U_V0);
    const double* Ts = sm + ((s & 1) ? S::U_T1 : S::U_T0);
    double* top = (MODE == GE) ? nullptr : topt + size_t(col0) * NB + b * IB;
    warp_apply<NB, TRANST>(x, r0 / 8, r1 / 8, Vs, Ts, top, lane);
    __syncthreads();
  }
  store_x<NB>(x, xt + size_t(col0) * NB, 0, NB / 8, lane);
}

// ---------------------------------------------------------------------------
// panel item: Householder QR of one tile (GE), of [R_piv; R_i] (TT) or of
// [R_piv; A_i] (TS), ib columns at a time: level-2 sweep of the block in
// shared memory (warp-shuffle reductions), T_b from the Gram matrix, then
// the block reflector applied to the trailing columns on DMMA.

template <int NB, int MODE>
__device__ void panel_item(double* sm, double* at /*GE: tile; TT/TS: bottom tile (i,k)*/,
                           double* rt /*TT/TS: pivot tile (piv,k)*/, double* tslot, int tid) {
  using S = Smem<NB>;
  constexpr int PLD = S::PLD;
  const int warp = tid >> 5, lane = tid & 31;
  double* P = sm + S::P_P;
  double* Vs = sm + S::P_V;
  double* Ts = sm + S::P_T;
  double* G = sm + S::P_G;
  double* tau_s = sm + S::P_SC;
  double* scal_s = tau_s + IB;
  double* beta_s = tau_s + 2 * IB;
  double* nrm2_s = tau_s + 3 * IB;

  for (int b = 0; b < NB / IB; ++b) {
    const int rb0 = b * IB;
    // rows of the stacked panel and the vector rows of column j
    const int nrow = (MODE == GE) ? NB - rb0 : (MODE == TT ? IB + rb0 + IB : IB + NB);
    auto vlo = [&](int j) { return MODE == GE ? j + 1 : IB; };
    auto vhi = [&](int j) { return MODE == GE ? nrow : (MODE == TT ? IB + rb0 + j + 1 : nrow); };

    // ---- load the panel block into P
    if (MODE == GE) {
      for (int e = tid; e < nrow * IB; e += NT) {
        const int pr = e % nrow, j = e / nrow;
        P[pr + j * PLD] = __ldcg(at + (rb0 + pr) + size_t(rb0 + j) * NB);
      }
    } else {
      for (int e = tid; e < IB * IB; e += NT) {
        const int r = e % IB, j = e / IB;
        P[r + j * PLD] = (r <= j) ? __ldcg(rt + (rb0 + r) + size_t(rb0 + j) * NB) : 0.0;
      }
      const int nb_rows = nrow - IB;
      for (int e = tid; e < nb_rows * IB; e += NT) {
        const int rr = e % nb_rows, j = e / nb_rows;
        double v = 0.0;
        if (MODE == TS || rr <= rb0 + j) v = __ldcg(at + rr + size_t(rb0 + j) * NB);
        P[IB + rr + j * PLD] = v;
      }
    }
    __syncthreads();
    // norm^2 of column 0 over its vector rows
    if (warp == 0) {
      double s = 0.0;
      for (int r = vlo(0) + lane; r < vhi(0); r += 32) s += P[r] * P[r];
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) nrm2_s[0] = s;
    }
    // ---- level-2 Householder sweep over the ib columns (dgeqr2 / dtpqrt2)
    for (int j = 0; j < IB; ++j) {
      __syncthreads();
      const double alpha = P[j + j * PLD];
      const double xn2 = nrm2_s[j];
      double tau = 0.0, scal = 0.0, beta = alpha;
      if (xn2 != 0.0) {
        beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      if (tid == 0) {
        tau_s[j] = tau;
        scal_s[j] = scal;
        beta_s[j] = beta;
      }
      const int lo = vlo(j), hi = vhi(j);
      const double* vj = P + j * PLD;
      // columns c = j+1.. handled by warp (c % NW)
      int c = j + 1 + ((warp - (j + 1)) % NW + NW) % NW;
      for (; c < IB; c += NW) {
        double* pc = P + c * PLD;
        if (tau != 0.0) {
          double d = 0.0;
          for (int r = lo + lane; r < hi; r += 32) d += vj[r] * pc[r];
#pragma unroll
          for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          const double s = tau * (pc[j] + scal * d);
          const double sv = s * scal;
          for (int r = lo + lane; r < hi; r += 32) pc[r] -= sv * vj[r];
          __syncwarp();
          if (lane == 0) pc[j] -= s;
        }
        if (c == j + 1) {
          __syncwarp();
          double s2 = 0.0;
          for (int r = vlo(c) + lane; r < vhi(c); r += 32) s2 += pc[r] * pc[r];
#pragma unroll
          for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
          if (lane == 0) nrm2_s[c] = s2;
        }
      }
    }
    __syncthreads();
    // scale the reflectors, put beta on the diagonal
    for (int e = tid; e < nrow * IB; e += NT) {
      const int pr = e % nrow, j = e / nrow;
      if (pr >= vlo(j) && pr < vhi(j) && tau_s[j] != 0.0) P[pr + j * PLD] *= scal_s[j];
      if (pr == j) P[pr + j * PLD] = beta_s[j];
    }
    __syncthreads();
    // ---- Gram matrix of the block's reflectors: G[i][j] = v_i . v_j (i < j)
    for (int pidx = warp; pidx < IB * IB; pidx += NW) {
      const int i = pidx % IB, j = pidx / IB;
      if (i >= j) continue;
      const double* vi = P + i * PLD;
      const double* vjj = P + j * PLD;
      double d = 0.0;
      const int lo = vlo(j), hi = (MODE == TT) ? vhi(i) : vhi(j);
      for (int r = lo + lane; r < hi; r += 32) d += vi[r] * vjj[r];
#pragma unroll
      for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      if (lane == 0) G[i + j * IB] = d + (MODE == GE ? vi[j] : 0.0);
    }
    __syncthreads();
    // ---- T_b by the dlarft recurrence: lane i owns row i of T
    if (warp == 0) {
      const int i = lane;
      double trow[IB];
#pragma unroll
      for (int j = 0; j < IB; ++j) trow[j] = 0.0;
#pragma unroll
      for (int j = 0; j < IB; ++j) {
        const double tj = tau_s[j];
        if (i == j) trow[j] = tj;
        if (i < j) {
          double s = 0.0;
#pragma unroll
          for (int l = 0; l < IB; ++l)
            if (l >= i && l < j) s += trow[l] * G[l + j * IB];
          trow[j] = -tj * s;
        }
      }
#pragma unroll
      for (int j = 0; j < IB; ++j) {
        Ts[swz(i, j)] = trow[j];
        tslot[i + size_t(rb0 + j) * IB] = trow[j];
      }
    }
    // ---- stage V for the trailing update, write the block back to HBM
    const int vrows0 = (MODE == GE) ? rb0 : 0;
    const int vrows1 = (MODE == GE) ? NB : (MODE == TT ? rb0 + IB : NB);
    for (int e = tid; e < (vrows1 - vrows0) * IB; e += NT) {
      const int rr = vrows0 + e % (vrows1 - vrows0), j = e / (vrows1 - vrows0);
      const int col = rb0 + j;
      double v;
      if (MODE == GE) {
        const int pr = rr - rb0;
        v = (pr > j) ? P[pr + j * PLD] : (pr == j ? 1.0 : 0.0);
        at[rr + size_t(col) * NB] = P[pr + j * PLD];
      } else {
        const bool live = (MODE == TS) || (rr <= col);
        v = live ? P[IB + rr + j * PLD] : 0.0;
        if (live) at[rr + size_t(col) * NB] = v;
      }
      Vs[swz(rr, j)] = v;
    }
    if (MODE != GE) {
      for (int e = tid; e < IB * IB; e += NT) {
        const int r = e % IB, j = e / IB;
        if (r <= j) rt[(rb0 + r) + size_t(rb0 + j) * NB] = P[r + j * PLD];
      }
    }
    __syncthreads();
    // ---- trailing update of columns rb0+IB .. NB on DMMA, 8 columns per warp
    const int nch = (NB - rb0 - IB) / 8;
    const int g0 = (MODE == GE) ? rb0 / 8 : 0;
    const int g1 = (MODE == TT) ? (rb0 + IB) / 8 : NB / 8;
    for (int ch = warp; ch < nch; ch += NW) {
      const int col = rb0 + IB + ch * 8;
      double x[NB / 8][2];
      load_x<NB>(x, at + size_t(col) * NB, g0, g1, lane);
      double* top = (MODE == GE) ? nullptr : rt + size_t(col) * NB + rb0;
      warp_apply<NB, true>(x, g0, g1, Vs, Ts, top, lane);
      store_x<NB>(x, at + size_t(col) * NB, g0, g1, lane);
    }
    __syncthreads();
  }
}

}  // namespace tqrk
