// Microbenchmark of the update work item in isolation: every CTA (one per SM)
// runs `reps` UNMQR/TTMQR slab items on private tiles (no dependencies).
// Reports per-item microseconds and the DMMA-pipe fraction of the FP64 peak.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1303_3182_b200/csrc/tqr_tasks.cuh"

using namespace tqrk;

template <int NB, int MODE>
__global__ void __launch_bounds__(NTP, 1) k_upd(double* tiles, double* tt, int reps) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) unsigned long long bars[4];
  unsigned seq = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 2 * 32 * NPW);
    mbar_init(&bars[1], 2 * 32 * NPW);
    mbar_init(&bars[2], NW);
    mbar_init(&bars[3], NW);
  }
  __syncthreads();
  const size_t T2 = size_t(NB) * NB;
  double* base = tiles + size_t(blockIdx.x) * 3 * T2;  // V tile, X tile, top tile
  const int warp = threadIdx.x >> 5;
  if (warp >= NW) {
    setmaxnreg_dec<40>();
    for (int r = 0; r < reps; ++r) {
      if (threadIdx.x == NT + 32) {  // the executor prefetches the next item's data tiles into L2
        const int ns = (r + 1) % (NB / WS);
        prefetch_l2(base + T2 + size_t(ns) * WS * NB, WS * NB * 8);
        prefetch_l2(base + 2 * T2 + size_t(ns) * WS * NB, WS * NB * 8);
      }
#ifndef TQR_ABL_NOPROD
      update_produce<NB, MODE, true>(sm, base, tt, base + 2 * T2, r % (NB / WS), warp - NW, threadIdx.x & 31, bars,
                                     bars + 2, seq);
#endif
      seq += NB / IB;
      bar_all();
    }
    return;
  }
  setmaxnreg_inc<232>();
  for (int r = 0; r < reps; ++r) {
    update_consume<NB, MODE, true>(sm, base + T2, base + 2 * T2, r % (NB / WS), threadIdx.x, bars, bars + 2, seq);
    seq += NB / IB;
    bar_all();
  }
}

template <int NB, int MODE>
void run(const char* name, int sms) {
  const size_t T2 = size_t(NB) * NB;
  double *tiles, *tt;
  cudaMalloc(&tiles, sms * 3 * T2 * sizeof(double));
  cudaMalloc(&tt, IB * NB * sizeof(double));
  std::vector<double> h(sms * 3 * T2);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 1e-3 * double((i * 7919) % 1000) / 1000.0;
  cudaMemcpy(tiles, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  std::vector<double> ht(IB * NB, 0.01);
  cudaMemcpy(tt, ht.data(), ht.size() * 8, cudaMemcpyHostToDevice);
  auto k = k_upd<NB, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Smem<NB>::BYTES));
  const int reps = 64;
  k<<<sms, NTP, Smem<NB>::BYTES>>>(tiles, tt, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<sms, NTP, Smem<NB>::BYTES>>>(tiles, tt, reps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double us = ms * 1e3 / reps;
  // DMMAs per warp per item (incl. T multiply): sum over blocks
  long dm = 0;
  for (int bb = 0; bb < NB / IB; ++bb) {
    int rows = MODE == GE ? NB - bb * IB : (MODE == TT ? (bb + 1) * IB : NB);
    dm += 2 * (rows / 8) * 8 + 20;
  }
  const double dmma_flops = double(dm) * 8 * 512 * sms * reps;
  const double useful = 2.0 * NB * NB * WS * (MODE == TS ? 2.0 : 1.0) * sms * reps;
#ifdef TQR_PROF_UPD
  unsigned long long hp[32];
  cudaMemcpyFromSymbol(hp, g_uprof, sizeof(hp));
  unsigned long long zero[32] = {0};
  cudaMemcpyToSymbol(g_uprof, zero, sizeof(zero));
  for (int i = 16; i < 32; ++i) hp[0] += hp[i];
  double tot = double(hp[0] + hp[2] + hp[6] + hp[8]);
  printf("phases (frac): load_x %.3f wait_full %.3f apply %.3f store %.3f\n", hp[8] / tot, hp[0] / tot, hp[2] / tot,
         hp[6] / tot);
  {
    const double nbw = 8.0 * sms * (reps + 4) * (NB / IB);  // warp-blocks
    printf("cycles per warp-block: gemm1 issue %.0f drain %.0f | combine+T issue %.0f drain %.0f | gemm2 issue %.0f drain %.0f | total apply %.0f\n",
           hp[10] / nbw, hp[13] / nbw, hp[14] / nbw, hp[11] / nbw, hp[15] / nbw, hp[12] / nbw, hp[2] / nbw);
  }
  printf("producer per warp-item: wait empty %.0f issue %.0f\n", hp[3] / (4.0 * 148 * 68), hp[4] / (4.0 * 148 * 68));
  printf("wait_full per block:");
  for (int i = 0; i < 8; ++i) printf(" %.0f", (hp[16 + i] + hp[24 + i]) / (8.0 * 148 * 68));
  printf("\n");
#endif
  printf("{\"item\": \"%s\", \"nb\": %d, \"us_per_item\": %.2f, \"dmma_tflops\": %.2f, \"useful_tflops\": %.2f, \"err\": \"%s\"}\n",
         name, NB, us, dmma_flops / (ms * 1e-3) / 1e12, useful / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(tiles);
  cudaFree(tt);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<256, GE>("UNMQR", sms);
  run<256, TT>("TTMQR", sms);
  run<256, TS>("TSMQR", sms);
  run<64, GE>("UNMQR", sms);
  run<64, TT>("TTMQR", sms);
  return 0;
}
