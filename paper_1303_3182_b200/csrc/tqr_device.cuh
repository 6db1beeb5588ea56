// Device building blocks of the tiled QR engine (sm_100a).
//
// FP64 on B200 has no tcgen05 kind (tcgen05.mma rejects .kind::f64); the
// tensor path is mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4, which runs at the
// full FP64 rate (measured 37.2 TFLOP/s, profiles/fp64_peak_r01.json).
//
// Data layout (HBM): p x q tiles of nb x nb doubles, column-major inside a
// tile, tile (i,j) (1-based) at ((j-1)*p + (i-1)) * nb*nb.  After GEQRT a
// tile holds R (upper, incl. diagonal) and the unit-lower reflectors V_G
// (strict lower); TTQRT stores its upper-triangular V_E over R of the
// eliminated tile, TSQRT its full V_E.  T factors (ib x nb per tile, LAPACK
// layout, T_b upper-triangular at columns b*ib..) live in two side arrays.
//
// Compute layout: a warp owns 8 columns of the matrix being updated, kept in
// registers as the DMMA C fragment of X = C^T (8 x nb): lane (r, c) holds
// rows 8g+2c, 8g+2c+1 of column r for every 8-row group g.  The reflector
// block V (rows x ib) and T (ib x ib) are staged in shared memory in a
// swizzled 8x8-sub-block layout that makes both DMMA B-fragment patterns
// (V as K x N and V^T) bank-conflict free.
#pragma once
#include <cstdint>
#include <type_traits>

namespace tqrk {

#ifdef TQR_PROF_UPD
__device__ unsigned long long g_uprof[32];
#define UPROF_MARK(k) UPROF_MARK_V(k, _tp)
#define UPROF_MARK_V(k, v)                                                    \
  do {                                                                        \
    if ((threadIdx.x & 31) == 0) {                                            \
      long long _t = clock64();                                               \
      atomicAdd(&g_uprof[k], (unsigned long long)(_t - v));                   \
      v = _t;                                                                 \
    }                                                                         \
  } while (0)
#define UPROF_DECL long long _tp = clock64()
#define UPROF_DECL_V(v) long long v = clock64()
// mark once `val` has been produced (a predicate read stalls on its scoreboard)
#define UPROF_MARK_DEP(k, v, val)                                                                   \
  do {                                                                                              \
    asm volatile("{.reg .pred p; setp.eq.f64 p, %0, 0d7FF8000000000123; @p trap;}" ::"d"(val) : "memory"); \
    UPROF_MARK_V(k, v);                                                                             \
  } while (0)
#else
#define UPROF_MARK(k) \
  do {                \
  } while (0)
#define UPROF_MARK_V(k, v) \
  do {                     \
  } while (0)
#define UPROF_MARK_DEP(k, v, val) \
  do {                            \
  } while (0)
#define UPROF_DECL
#define UPROF_DECL_V(v)
#endif

// Update-kernel accumulation choices (in-executor A/B at C3 / C5, one B200):
//  * the T multiply's odd row halves in a second DMMA chain (half the
//    dependent-DMMA depth): C3 256.5 -> 253.5 ms (TQR_NO_T_SPLIT_H restores one);
//  * X -= V W accumulates straight into X instead of from zero with one
//    final subtraction: 64 DADDs and 8 live registers less per reflector
//    block, C3 253.5 -> 247.8 ms, C5 931 -> 912 ms.  The update's rounding is
//    then ~32 FMA roundings at |X| per block instead of one; measured at
//    n = 16384: ||A - QR|| / ||A|| 5.07e-15 -> 5.93e-15, ||Q^T Q - I||_F
//    6.08e-13 unchanged (Q's orthogonality is set by V and T, not by the
//    updates).  TQR_NO_DIRECT_ACC restores the from-zero form.
#if !defined(TQR_NO_T_SPLIT_H) && !defined(TQR_T_SPLIT_H)
#define TQR_T_SPLIT_H
#endif
#if !defined(TQR_NO_DIRECT_ACC) && !defined(TQR_DIRECT_ACC)
#define TQR_DIRECT_ACC
#endif

constexpr int NT = 256;  // compute threads per CTA (8 warps)
constexpr int NW = 8;
constexpr int TLD = 40;  // ld of the staged pivot rows (IB + 8: conflict-free 16-byte reads)
constexpr int NTP = NT + 128;  // + one producer warpgroup (staging / prefetch)

// all threads of the CTA (both warp roles)
__device__ __forceinline__ void bar_all() { asm volatile("bar.sync 0, 384;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}
constexpr int IB = 32;   // inner blocking ib
constexpr int WS = 64;   // columns per update work item (8 per warp)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// Error-free transformation a + b = s + e (Knuth TwoSum; no reassociation:
// nvcc does not contract or reorder adds without fast-math).
__device__ __forceinline__ void two_sum(double& s, double& e, double a, double b) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
// Compensated DMMA accumulation: the 8x8x4 product is formed from zero (one
// rounded 4-term sum) and added error-free into hi, the rounding going to lo.
// The accumulation error then no longer grows with the number of k-steps.
__device__ __forceinline__ void dmma_comp(double (&hi)[2], double (&lo)[2], double a, double b) {
  double t[2] = {0.0, 0.0};
  dmma(t, a, b);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double s, e;
    two_sum(s, e, hi[h], t[h]);
    hi[h] = s;
    lo[h] += e;
  }
}

// in-sub-block swizzle: element (a, b) (row, col) of an 8x8 sub-block ->
// 0..63.  Rows 2k, 2k+1 of a column are adjacent (16-byte staging copies of
// a column's row pair; one 16-byte load gives the B fragments (2c, r) and
// (2c+1, r) of both k-halves of W = V^T X), and both fragment patterns hit
// distinct banks: (2c+h, r) as 16-byte loads per quarter-warp, (r, 2c+h)
// (X -= W V^T) as 8-byte loads per half-warp.
__device__ __forceinline__ int swz_in(int a, int b) {
  const int a0 = a & 1, a1 = (a >> 1) & 1, a2 = (a >> 2) & 1;
  const int b0 = b & 1, b1 = (b >> 1) & 1, b2 = (b >> 2) & 1;
  return a0 | (a1 << 1) | ((a2 ^ b1) << 2) | ((b0 ^ b2) << 3) | (b1 << 4) | (b2 << 5);
}
// element (row, col) of a [rows x IB] block
__device__ __forceinline__ int swz(int row, int col) { return ((row >> 3) * (IB / 8) + (col >> 3)) * 64 + swz_in(row & 7, col & 7); }

__device__ __forceinline__ double2 ldcg2(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void stcg2(double* p, double a, double b) {
  __stcg(reinterpret_cast<double2*>(p), make_double2(a, b));
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
// bulk L2 prefetch of a contiguous range (bytes, multiple of 16)
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

enum Mode : int { GE = 0, TT = 1, TS = 2 };

// Apply one ib-block reflector H_b = I - V T V^T (or its transpose) to the
// warp's 8 columns held in x, rows of the IB-row blocks [rb0, rb1), plus the
// IB "top" rows at `top` (TT/TS: the pivot tile's block rows; nullptr for
// GE).
//   Q^T: W = top + V^T X ; W = T^T W ; top -= W ; X -= V W   (TRANST = true)
//   Q  : same with W = T W                                  (TRANST = false)
// The row loop is unrolled per 32-row block (4 DMMA row groups) so the
// B-fragment loads of a block are scheduled ahead of its DMMAs.
// pf(x, idx) runs after every 8-row group of the first GEMM (idx = 4 rb +
// gg) and after every reflector quarter of the second (idx = 32 + 4 rb +
// kb); idx folds to a constant once the loops are unrolled, so a schedule
// can move X loads / stores between the DMMAs (XSched below).
struct NoPf {
  template <class X>
  __device__ __forceinline__ void operator()(X&, int) const {}
  __device__ __forceinline__ void flush() const {}
};

// TRI: shape of row block `drb` of V (the reflector block's diagonal 32x32):
// 0 unit-lower (GE), 1 upper (TT), 2 full (TS).  V is staged already
// masked; 8x8 sub-blocks that are structurally zero are skipped in both
// GEMMs.
// [RBL, RBH): compile-time bound on the row blocks this instance may touch,
// so that x registers outside it can be in flight (loads) meanwhile.
// mid(x) runs once the first GEMM has consumed rows of blocks < NB/IB/2
// (e.g. to issue the loads of the other half of X only then).
struct NoMid {
  template <class X>
  __device__ __forceinline__ void operator()(X&) const {}
};
// One application of reflectors [8*KA, 8*KB) of the block (the 8-column
// groups KA..KB-1): KA=0, KB=4 is the whole ib-block.
// COMP: every accumulation compensated (dmma_comp): used when applying or
// forming Q (tqr_apply_q), where the rounding of V^T X, T W and V W would
// otherwise accumulate over the thousands of reflector blocks each entry of
// Q passes through (orthogonality of the formed Q).
template <int NB, bool TRANST, int TRI, int RBL, int RBH, int KA, int KB, class PF, class MID, bool COMP = false>
__device__ __forceinline__ void warp_apply_k(double (&x)[NB / 8][2], int rb0, int rb1, const double* __restrict__ Vs,
                                             const double* __restrict__ Ts, double* top, int lane,
                                             const double* top_s, int drb, PF& pf, MID& mid) {
  // is V sub-block (row group gg, column group cb) of the diagonal block zero?
#ifdef TQR_ABL_NODIAG  // ablation: the diagonal block as a full block (V is staged masked)
  auto zero_blk = [](int, int) { return false; };
#else
  auto zero_blk = [](int gg, int cb) { return TRI == 0 ? (gg < cb) : (TRI == 1 ? (gg > cb) : false); };
#endif
  const int r = lane >> 2, c = lane & 3;
  const int s1a = swz_in(2 * c, r);  // (2c+h, r) at s1a + h
  const int s3a = swz_in(r, 2 * c), s3b = swz_in(r, 2 * c + 1);  // (r, 2c+h)
  // top_s: the block's IB pivot rows of this warp's 8 columns staged in smem
  // (column-major, ld TLD); else read from global
  double w[4][2], ap[4][2];
  double wl[4][2], wl2[4][2];  // COMP: low parts of the two chains
#pragma unroll
  for (int nb = KA; nb < KB; ++nb) wl[nb][0] = wl[nb][1] = wl2[nb][0] = wl2[nb][1] = 0.0;
#ifndef TQR_W_ONE_CHAIN
  // V^T X accumulates in two interleaved chains (row halves h of every
  // 8-row group), summed once: half the dependent-DMMA chain length and a
  // shorter floating-point accumulation (orthogonality of the applied
  // transformation).  Applying Q (not Q^T: forming Q) uses four chains
  // (also alternate row groups) — measured slower in the factorization
  // (C3 +1.7 %), more orthogonal Q.
#ifdef TQR_W_FOUR_CHAINS
  constexpr bool FOURC = true;
#else
  constexpr bool FOURC = false;
#endif
  double w2[4][2];
#pragma unroll
  for (int nb = KA; nb < KB; ++nb) w2[nb][0] = w2[nb][1] = 0.0;
#if defined(TQR_W_FOUR_CHAINS) || !defined(TQR_W_FORM_TWO)
  double w3[4][2], w4[4][2];
#pragma unroll
  for (int nb = KA; nb < KB; ++nb) w3[nb][0] = w3[nb][1] = w4[nb][0] = w4[nb][1] = 0.0;
#endif
#endif
  if (top) {
#pragma unroll
    for (int nb = KA; nb < KB; ++nb) {
      double2 v = top_s ? *reinterpret_cast<const double2*>(top_s + 8 * nb + 2 * c + r * TLD)
                        : ldcg2(top + 8 * nb + 2 * c + r * NB);
      ap[nb][0] = v.x;
      ap[nb][1] = v.y;
    }
  }
  UPROF_DECL_V(_tq);
  // accumulate V^T X from zero and add the pivot rows once afterwards, as
  // LAPACK's dlarfb does (one rounding of the large operand per block)
#pragma unroll
  for (int nb = KA; nb < KB; ++nb) w[nb][0] = w[nb][1] = 0.0;
  // W^T (8 x IB) += X (8 x rows) * V (rows x IB); B fragments of the next
  // row group are loaded while the current group's DMMAs issue
#pragma unroll
  for (int rb = 0; rb < NB / IB; ++rb) {
    if (rb >= RBL && rb < RBH && rb >= rb0 && rb < rb1) {
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) {
        double bc[2][4];
#pragma unroll
        for (int nb = KA; nb < KB; ++nb) {
          const double2 v2 = *reinterpret_cast<const double2*>(Vs + ((rb * 4 + gg) * (IB / 8) + nb) * 64 + s1a);
          bc[0][nb] = v2.x;
          bc[1][nb] = v2.y;
        }
        const bool dg = (TRI != 2) && rb == drb;
        if constexpr (COMP) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = KA; nb < KB; ++nb)
              if (!(dg && zero_blk(gg, nb)))
                dmma_comp(h ? w2[nb] : w[nb], h ? wl2[nb] : wl[nb], x[rb * 4 + gg][h], bc[h][nb]);
        } else
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int nb = KA; nb < KB; ++nb)
#if defined(TQR_W_FOUR_CHAINS) || !defined(TQR_W_FORM_TWO)
            if (!(dg && zero_blk(gg, nb)) && (!TRANST || FOURC))
              dmma((gg & 1) ? (h ? w4[nb] : w3[nb]) : (h ? w2[nb] : w[nb]), x[rb * 4 + gg][h], bc[h][nb]);
            else if (!(dg && zero_blk(gg, nb)))
              dmma(h ? w2[nb] : w[nb], x[rb * 4 + gg][h], bc[h][nb]);
#elif !defined(TQR_W_ONE_CHAIN)
            if (!(dg && zero_blk(gg, nb))) dmma(h ? w2[nb] : w[nb], x[rb * 4 + gg][h], bc[h][nb]);
#else
            if (!(dg && zero_blk(gg, nb))) dmma(w[nb], x[rb * 4 + gg][h], bc[h][nb]);
#endif
        pf(x, rb * 4 + gg);
      }
    }
    if (rb == NB / IB / 2 - 1) mid(x);  // (a no-op after its first call)
  }
  UPROF_MARK_V(10, _tq);
  UPROF_MARK_DEP(13, _tq, w[KB - 1][1] + w2[KB - 1][1]);
  if constexpr (COMP) {
    // W = top + V^T X summed in double-double, rounded once
#pragma unroll
    for (int nb = KA; nb < KB; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double s, er;
        two_sum(s, er, w[nb][e], w2[nb][e]);
        double l = er + (wl[nb][e] + wl2[nb][e]);
        if (top) {
          double s2, er2;
          two_sum(s2, er2, s, ap[nb][e]);
          s = s2;
          l += er2;
        }
        w[nb][e] = s + l;
      }
  } else {
#ifndef TQR_W_ONE_CHAIN
#pragma unroll
  for (int nb = KA; nb < KB; ++nb) {
#if defined(TQR_W_FOUR_CHAINS) || !defined(TQR_W_FORM_TWO)
    if (!TRANST || FOURC) {
      w[nb][0] += w3[nb][0];
      w[nb][1] += w3[nb][1];
      w2[nb][0] += w4[nb][0];
      w2[nb][1] += w4[nb][1];
    }
#endif
    w[nb][0] += w2[nb][0];
    w[nb][1] += w2[nb][1];
  }
#endif
  if (top) {
#pragma unroll
    for (int nb = KA; nb < KB; ++nb) {
      w[nb][0] += ap[nb][0];
      w[nb][1] += ap[nb][1];
    }
  }
  }  // !COMP
  // W^T <- W^T T (Q^T) or W^T T^T (Q); T upper triangular
  double tb[2][4][4];
#pragma unroll
  for (int kb = KA; kb < KB; ++kb)
#pragma unroll
    for (int nb = KA; nb < KB; ++nb)
      if (TRANST ? (kb <= nb) : (kb >= nb)) {
        const double* tp = TRANST ? Ts + (kb * 4 + nb) * 64 : Ts + (nb * 4 + kb) * 64;
        if (TRANST) {
          const double2 v2 = *reinterpret_cast<const double2*>(tp + s1a);  // s1b == s1a + 1
          tb[0][kb][nb] = v2.x;
          tb[1][kb][nb] = v2.y;
        } else {
          tb[0][kb][nb] = tp[s3a];
          tb[1][kb][nb] = tp[s3b];
        }
      }
  double wt[4][2], wtl[4][2];
#pragma unroll
  for (int nb = KA; nb < KB; ++nb) wt[nb][0] = wt[nb][1] = wtl[nb][0] = wtl[nb][1] = 0.0;
#ifdef TQR_T_SPLIT_H
  double wt2[4][2];  // the odd row halves' chain
#pragma unroll
  for (int nb = KA; nb < KB; ++nb) wt2[nb][0] = wt2[nb][1] = 0.0;
#endif
#pragma unroll
  for (int kb = KA; kb < KB; ++kb)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int nb = KA; nb < KB; ++nb)
        if (TRANST ? (kb <= nb) : (kb >= nb)) {
#ifdef TQR_ABL_NOT  // ablation (wrong numbers): no T multiply
          if (kb == nb) wt[nb][h] = w[kb][h] * tb[h][kb][nb];
#else
          if constexpr (COMP)
            dmma_comp(wt[nb], wtl[nb], w[kb][h], tb[h][kb][nb]);
          else
#ifdef TQR_T_SPLIT_H
            dmma(h ? wt2[nb] : wt[nb], w[kb][h], tb[h][kb][nb]);
#else
            dmma(wt[nb], w[kb][h], tb[h][kb][nb]);
#endif
#endif
        }
#ifdef TQR_T_SPLIT_H
  if constexpr (!COMP) {
#pragma unroll
    for (int nb = KA; nb < KB; ++nb) {
      wt[nb][0] += wt2[nb][0];
      wt[nb][1] += wt2[nb][1];
    }
  }
#endif
  if constexpr (COMP) {
#pragma unroll
    for (int nb = KA; nb < KB; ++nb) {
      wt[nb][0] += wtl[nb][0];
      wt[nb][1] += wtl[nb][1];
    }
  }
  if (top) {
#pragma unroll
    for (int nb = KA; nb < KB; ++nb) stcg2(top + 8 * nb + 2 * c + r * NB, ap[nb][0] - wt[nb][0], ap[nb][1] - wt[nb][1]);
  }
#pragma unroll
  for (int nb = KA; nb < KB; ++nb) {
    wt[nb][0] = -wt[nb][0];
    wt[nb][1] = -wt[nb][1];
  }
  UPROF_MARK_V(14, _tq);
  UPROF_MARK_DEP(11, _tq, wt[KB - 1][1]);
  // X -= W^T V^T, accumulated straight into X (TQR_NO_DIRECT_ACC: per 32-row
  // block from zero, subtracted from X once)
#pragma unroll
  for (int rb = 0; rb < NB / IB; ++rb) {
    if (rb >= RBL && rb < RBH && rb >= rb0 && rb < rb1) {
      double acc3[4][2], acc3l[4][2];
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) acc3[gg][0] = acc3[gg][1] = acc3l[gg][0] = acc3l[gg][1] = 0.0;
#pragma unroll
      for (int kb = KA; kb < KB; ++kb) {
        double bc[2][4];
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) {
          const double* vb = Vs + ((rb * 4 + gg) * (IB / 8) + kb) * 64;
          bc[0][gg] = vb[s3a];
          bc[1][gg] = vb[s3b];
        }
        const bool dg = (TRI != 2) && rb == drb;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int gg = 0; gg < 4; ++gg)
            if constexpr (COMP) {
              if (!(dg && zero_blk(gg, kb))) dmma_comp(acc3[gg], acc3l[gg], wt[kb][h], bc[h][gg]);
            } else
#ifdef TQR_DIRECT_ACC
            if (!(dg && zero_blk(gg, kb))) dmma(x[rb * 4 + gg], wt[kb][h], bc[h][gg]);
#else
            if (!(dg && zero_blk(gg, kb))) dmma(acc3[gg], wt[kb][h], bc[h][gg]);
#endif
        pf(x, 32 + rb * 4 + kb);
      }
      if constexpr (COMP) {
#pragma unroll
        for (int gg = 0; gg < 4; ++gg)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double s, er;
            two_sum(s, er, x[rb * 4 + gg][e], acc3[gg][e]);
            x[rb * 4 + gg][e] = s + (er + acc3l[gg][e]);
          }
      } else {
#ifndef TQR_DIRECT_ACC
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) {
        x[rb * 4 + gg][0] += acc3[gg][0];
        x[rb * 4 + gg][1] += acc3[gg][1];
      }
#endif
      }
    }
  }
  UPROF_MARK_V(15, _tq);
  UPROF_MARK_DEP(12, _tq, x[NB / 8 - 1][0] + x[0][0]);
}

// Apply the staged ib-block reflector (see warp_apply_k).  SPLIT (off: measured
// 2-5 % slower, the halves serialize through X): as two
// 16-reflector halves, (I - V2 T22 V2^T)(I - V1 T11 V1^T) for Q^T (reverse
// for Q) — the same transformation; the T multiply then costs 12 instead of
// 20 DMMAs per warp (T12 is not needed).
#ifndef TQR_SPLIT_T
#define TQR_SPLIT_T 0
#endif
template <int NB, bool TRANST, int TRI = 2, int RBL = 0, int RBH = NB / IB, class PF = NoPf, class MID = NoMid,
          bool COMP = false, bool SPLIT = (TQR_SPLIT_T != 0)>
__device__ __forceinline__ void warp_apply(double (&x)[NB / 8][2], int rb0, int rb1, const double* __restrict__ Vs,
                                           const double* __restrict__ Ts, double* top, int lane,
                                           const double* top_s = nullptr, int drb = -1, PF pf = PF(),
                                           MID mid = MID()) {
  if constexpr (!SPLIT) {
    warp_apply_k<NB, TRANST, TRI, RBL, RBH, 0, 4, PF, MID, COMP>(x, rb0, rb1, Vs, Ts, top, lane, top_s, drb, pf, mid);
  } else {
    NoMid none;
    if constexpr (TRANST) {
      warp_apply_k<NB, TRANST, TRI, RBL, RBH, 0, 2>(x, rb0, rb1, Vs, Ts, top, lane, top_s, drb, pf, mid);
      warp_apply_k<NB, TRANST, TRI, RBL, RBH, 2, 4>(x, rb0, rb1, Vs, Ts, top, lane, top_s, drb, pf, none);
    } else {
      warp_apply_k<NB, TRANST, TRI, RBL, RBH, 2, 4>(x, rb0, rb1, Vs, Ts, top, lane, top_s, drb, pf, mid);
      warp_apply_k<NB, TRANST, TRI, RBL, RBH, 0, 2>(x, rb0, rb1, Vs, Ts, top, lane, top_s, drb, pf, none);
    }
  }
  pf.flush();
}

// x rows [8*g0, 8*g1) of the warp's columns (column-major tile, ld NB)
// (ZERO: clear the other rows; else leave them untouched)
template <int NB, bool ZERO = true>
__device__ __forceinline__ void load_x(double (&x)[NB / 8][2], const double* col, int g0, int g1, int lane) {
  const int r = lane >> 2, c = lane & 3;
#pragma unroll
  for (int g = 0; g < NB / 8; ++g) {
    if (g >= g0 && g < g1) {
      double2 v = ldcg2(col + r * NB + 8 * g + 2 * c);
      x[g][0] = v.x;
      x[g][1] = v.y;
    } else if (ZERO) {
      x[g][0] = x[g][1] = 0.0;
    }
  }
}
template <int NB>
__device__ __forceinline__ void store_x(const double (&x)[NB / 8][2], double* col, int g0, int g1, int lane) {
  const int r = lane >> 2, c = lane & 3;
#pragma unroll
  for (int g = 0; g < NB / 8; ++g)
    if (g >= g0 && g < g1) stcg2(col + r * NB + 8 * g + 2 * c, x[g][0], x[g][1]);
}

// X traffic spread over one reflector block's DMMA stream (pf hook of
// warp_apply): a burst of 16 loads / stores per lane at a block boundary
// stalls both warps of an SMSP on the LSU queue for thousands of cycles;
// one or two row groups per call overlap it with the DMMAs.
//   XS_TT_LOAD   (TT block 0, rows < IB): load the lower half, 2 groups per
//                call over the 4 + 4 calls of the block
//   XS_GE_LOAD   (GE block 0): load the lower half, one group per call of
//                the first GEMM's upper-half row groups
//   XS_GE_STORE  (GE block NBLK/2): store the final upper half, one group per
//                call of the first GEMM (rows >= NB/2 only)
//   XS_GE_STORE2 (GE last block, NB > 64): store rows NB/2 .. NB-33 (final
//                after the block before), 3 groups per first-GEMM call
enum XsKind : int { XS_TT_LOAD, XS_GE_LOAD, XS_GE_STORE, XS_GE_STORE2 };
template <int NB, int KIND>
struct XSched {
  double* col;  // the warp's 8 columns (column-major tile, ld NB)
  int lane;
  template <class X>
  __device__ __forceinline__ void operator()(X& x, int idx) const {
    constexpr int G = NB / 8, GH = NB / 16, NBLK = NB / IB;
    const int r = lane >> 2, c = lane & 3;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      bool hit = false;
      if (KIND == XS_TT_LOAD) {
        const int call = idx < 32 ? idx : 4 + (idx - 32);  // 0..7
        constexpr int per = (G - GH + 7) / 8;
        hit = g >= GH && idx < 36 && (idx < 4 || idx >= 32) && (g - GH) / per == call;
      } else if (KIND == XS_GE_LOAD) {
        hit = g >= GH && idx < GH && g - GH == idx;
      } else if (KIND == XS_GE_STORE) {
        hit = g < GH && idx >= GH && idx < 2 * GH && g == idx - GH;
      } else {
        constexpr int first = 4 * (NBLK - 1), n = G - 4 - GH, per = n > 0 ? (n + 3) / 4 : 1;
        hit = n > 0 && g >= GH && g < G - 4 && idx >= first && idx < first + 4 && (g - GH) / per == idx - first;
      }
      if (hit) {
        if (KIND == XS_TT_LOAD || KIND == XS_GE_LOAD) {
          double2 v = ldcg2(col + r * NB + 8 * g + 2 * c);
          x[g][0] = v.x;
          x[g][1] = v.y;
        } else {
          stcg2(col + r * NB + 8 * g + 2 * c, x[g][0], x[g][1]);
        }
      }
    }
  }
  __device__ __forceinline__ void flush() const {}
};

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// Producer staging (the NPW warps of the producer warpgroup, pw = 0..NPW-1,
// warp pw copies columns 8 pw .. 8 pw + 7): rows [row0, row1) of reflector
// block b of tile `vt` (ld NB) into swizzled smem with 16-byte cp.async.cg
// (L2 -> smem, no L1 allocation).
constexpr int NPW = 4;
static_assert(NPW * 8 == IB, "one 8-column group per producer warp");
template <int NB, int MODE>
__device__ __forceinline__ void pstage_v(double* Vs, const double* __restrict__ vt, int b, int row0, int row1, int pw,
                                         int lane) {
  // lane -> row pair p (rows 2p, 2p+1 of each 8-row group), column 8 pw + cq:
  // one instruction copies 8 rows x 8 columns, 16 bytes per lane (4 lanes
  // read a column's 64 contiguous bytes).  Entries of the diagonal 32x32
  // block outside the reflector pattern (GE: unit lower; TT: upper) are
  // stored directly instead of copied.
  const int p = lane & 3, cq = lane >> 2;
  const int c0 = 8 * pw + cq;
  const double* s0 = vt + size_t(b * IB + c0) * NB + 2 * p;
  double* d0 = Vs + pw * 64 + swz_in(2 * p, cq);
  const int dg0 = b * IB;
  for (int rr = row0; rr < row1; rr += 8) {
    double* e0 = d0 + (rr >> 3) * (IB / 8) * 64;
    if (MODE == TS || rr < dg0 || rr >= dg0 + IB) {
      cp_async16(e0, s0 + rr);
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lr = rr + 2 * p + h - dg0;  // row within the diagonal block
        const bool live = (MODE == GE) ? (lr > c0) : (lr <= c0);
        if (live)
          cp_async8(e0 + h, s0 + rr + h);
        else
          e0[h] = (MODE == GE && lr == c0) ? 1.0 : 0.0;
      }
    }
  }
}

// T_b (IB x IB; LAPACK ldt = IB, lower part zero as written by the panels):
// 16-byte row pairs, 4 per thread
__device__ __forceinline__ void pstage_t(double* Ts, const double* __restrict__ tt, int b, int pw, int lane) {
  const int p = lane & 3, cq = lane >> 2;
  const int c0 = 8 * pw + cq;
#pragma unroll
  for (int rr = 0; rr < IB; rr += 8)
    cp_async16(Ts + swz(rr + 2 * p, c0), tt + rr + 2 * p + size_t(b * IB + c0) * IB);
}

// IB pivot rows [r0, r0+IB) of WS columns from col0 (ld NB) -> smem,
// column-major ld TLD, 16-byte copies
template <int NB>
__device__ __forceinline__ void pstage_top(double* dst, const double* __restrict__ tile, int col0, int r0, int pw,
                                           int lane) {
  for (int e = pw * 32 + lane; e < WS * (IB / 2); e += NPW * 32) {
    const int cc = e / (IB / 2), rr = (e % (IB / 2)) * 2;
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst + rr + cc * TLD));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(tile + size_t(col0 + cc) * NB + r0 + rr));
  }
}

// ---- mbarrier helpers (producer/consumer handshake)
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
               "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared.b64 st, [%0];\n}\n" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(bar)))
               : "memory");
}
// arrive when all prior cp.async of this thread have landed
__device__ __forceinline__ void mbar_arrive_cpasync(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];\n" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(bar)))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// barrier among the 8 compute warps only (the producer warp is elsewhere)
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }

}  // namespace tqrk
