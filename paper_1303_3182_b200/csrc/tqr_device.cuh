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

namespace tqrk {

constexpr int NT = 256;  // threads per CTA (8 warps)
constexpr int NW = 8;
constexpr int IB = 32;   // inner blocking ib
constexpr int WS = 64;   // columns per update work item (8 per warp)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// in-sub-block swizzle: element (a, b) of an 8x8 sub-block -> 0..63 such that
// for lane (r,c): {(2c+h, r)} and {(r, 2c+h)} each hit 16 distinct 8-byte
// banks per half-warp.
__device__ __forceinline__ int swz_in(int a, int b) {
  const int a0 = a & 1, a1 = (a >> 1) & 1, a2 = (a >> 2) & 1;
  const int b0 = b & 1, b1 = (b >> 1) & 1, b2 = (b >> 2) & 1;
  return (a0 << 5) | (b2 << 4) | (a1 << 3) | (b1 << 2) | ((a2 ^ a0) << 1) | (b0 ^ b2);
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
// warp's 8 columns held in x (rows of groups [g0, g1)), plus the IB "top"
// rows at `top` (TT/TS: the pivot tile's block rows; nullptr for GE).
//   Q^T: W = top + V^T X ; W = T^T W ; top -= W ; X -= V W   (TRANST = true)
//   Q  : same with W = T W                                  (TRANST = false)
template <int NB, bool TRANST>
__device__ __forceinline__ void warp_apply(double (&x)[NB / 8][2], int g0, int g1, const double* __restrict__ Vs,
                                           const double* __restrict__ Ts, double* top, int lane) {
  const int r = lane >> 2, c = lane & 3;
  const int s1a = swz_in(2 * c, r), s1b = swz_in(2 * c + 1, r);  // (2c+h, r)
  const int s3a = swz_in(r, 2 * c), s3b = swz_in(r, 2 * c + 1);  // (r, 2c+h)
  double w[4][2], ap[4][2];
  if (top) {
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      double2 v = ldcg2(top + 8 * nb + 2 * c + r * NB);
      ap[nb][0] = v.x;
      ap[nb][1] = v.y;
      w[nb][0] = v.x;
      w[nb][1] = v.y;
    }
  } else {
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) w[nb][0] = w[nb][1] = ap[nb][0] = ap[nb][1] = 0.0;
  }
  // W^T (8 x IB) += X (8 x rows) * V (rows x IB)
#pragma unroll
  for (int g = 0; g < NB / 8; ++g) {
    if (g >= g0 && g < g1) {
      const double* vb = Vs + g * (IB / 8) * 64;
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) {
        dmma(w[nb], x[g][0], vb[nb * 64 + s1a]);
        dmma(w[nb], x[g][1], vb[nb * 64 + s1b]);
      }
    }
  }
  // W^T <- W^T T (Q^T) or W^T T^T (Q); T upper triangular
  double wt[4][2];
#pragma unroll
  for (int nb = 0; nb < 4; ++nb) wt[nb][0] = wt[nb][1] = 0.0;
#pragma unroll
  for (int kb = 0; kb < 4; ++kb)
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      if (TRANST ? (kb <= nb) : (kb >= nb)) {
        const double* tb = TRANST ? Ts + (kb * 4 + nb) * 64 : Ts + (nb * 4 + kb) * 64;
        dmma(wt[nb], w[kb][0], tb[TRANST ? s1a : s3a]);
        dmma(wt[nb], w[kb][1], tb[TRANST ? s1b : s3b]);
      }
    }
  if (top) {
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) stcg2(top + 8 * nb + 2 * c + r * NB, ap[nb][0] - wt[nb][0], ap[nb][1] - wt[nb][1]);
  }
#pragma unroll
  for (int nb = 0; nb < 4; ++nb) {
    wt[nb][0] = -wt[nb][0];
    wt[nb][1] = -wt[nb][1];
  }
  // X -= W^T V^T
#pragma unroll
  for (int g = 0; g < NB / 8; ++g) {
    if (g >= g0 && g < g1) {
      const double* vb = Vs + g * (IB / 8) * 64;
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
        dmma(x[g], wt[kb][0], vb[kb * 64 + s3a]);
        dmma(x[g], wt[kb][1], vb[kb * 64 + s3b]);
      }
    }
  }
}

// x rows [8*g0, 8*g1) of the warp's columns (column-major tile, ld NB)
template <int NB>
__device__ __forceinline__ void load_x(double (&x)[NB / 8][2], const double* col, int g0, int g1, int lane) {
  const int r = lane >> 2, c = lane & 3;
#pragma unroll
  for (int g = 0; g < NB / 8; ++g) {
    if (g >= g0 && g < g1) {
      double2 v = ldcg2(col + r * NB + 8 * g + 2 * c);
      x[g][0] = v.x;
      x[g][1] = v.y;
    } else {
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

// Stage block b of the reflectors of tile `vt` (ld NB) into swizzled smem,
// rows [row0, row1), masking per mode: GE unit-lower (diag block), TT
// upper-triangular, TS full.  Asynchronous (cp.async); masked entries are
// written directly.  All threads participate.
template <int NB, int MODE>
__device__ __forceinline__ void stage_v(double* Vs, const double* __restrict__ vt, int b, int row0, int row1, int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  const int a = lane & 7, cq = lane >> 3;
  const int col0 = b * IB;
  const int units = ((row1 - row0) >> 3) * (IB / 4);
  for (int u = warp; u < units; u += NW) {
    const int row = row0 + (u / (IB / 4)) * 8 + a;
    const int cl = (u % (IB / 4)) * 4 + cq;  // column within the block
    const int col = col0 + cl;
    double* dst = Vs + swz(row, cl);
    if (MODE == GE) {
      if (row > col)
        cp_async8(dst, vt + row + size_t(col) * NB);
      else
        *dst = (row == col) ? 1.0 : 0.0;
    } else if (MODE == TT) {
      if (row <= col)
        cp_async8(dst, vt + row + size_t(col) * NB);
      else
        *dst = 0.0;
    } else {
      cp_async8(dst, vt + row + size_t(col) * NB);
    }
  }
}

// Stage T_b (IB x IB upper triangular; LAPACK ldt = IB) into swizzled smem.
__device__ __forceinline__ void stage_t(double* Ts, const double* __restrict__ tt, int b, int tid) {
  for (int e = tid; e < IB * IB; e += NT) {
    const int row = e & (IB - 1), col = e / IB;  // row-fastest: coalesced
    double* dst = Ts + swz(row, col);
    if (row <= col)
      cp_async8(dst, tt + row + size_t(b * IB + col) * IB);
    else
      *dst = 0.0;
  }
}

}  // namespace tqrk
