// Microbenchmark of panel work items (GEQRT / TTQRT / TSQRT) in isolation:
// one CTA per SM, each factoring private tiles `reps` times.  Reports us per
// panel and the per-phase split (globaltimer, averaged over CTAs).
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_1303_3182_b200/csrc/tqr_tasks.cuh"

using namespace tqrk;

template <int NB, int MODE>
__global__ void __launch_bounds__(NTP, 1) k_pan(double* tiles, double* tslot, int reps, unsigned long long* prof) {
  extern __shared__ __align__(16) double sm[];
  const size_t T2 = size_t(NB) * NB;
  double* at = tiles + size_t(blockIdx.x) * 2 * T2;
  double* rt = at + T2;
  if (threadIdx.x >= NT) {
    setmaxnreg_dec<40>();
    return;
  }
  setmaxnreg_inc<232>();
  for (int r = 0; r < reps; ++r) {
    panel_run<NB, MODE>(sm, at, MODE == GE ? nullptr : rt, tslot + size_t(blockIdx.x) * IB * NB, threadIdx.x,
                         blockIdx.x == 0 ? prof : nullptr);
    csync();
  }
}

template <int NB, int MODE>
void run(const char* name, int sms) {
  const size_t T2 = size_t(NB) * NB;
  double *tiles, *ts;
  unsigned long long* prof;
  cudaMalloc(&tiles, sms * 2 * T2 * sizeof(double));
  cudaMalloc(&ts, sms * IB * NB * sizeof(double));
  cudaMalloc(&prof, 64 * 8);
  std::vector<double> h(sms * 2 * T2);
  unsigned long long s = 12345;
  for (auto& v : h) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    v = double((s >> 11) & 0xfffff) / double(0xfffff) - 0.5;
  }
  cudaMemcpy(tiles, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  auto k = k_pan<NB, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Smem<NB>::BYTES));
  const int reps = 4;
  cudaMemset(prof, 0, 64 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<sms, NTP, Smem<NB>::BYTES>>>(tiles, ts, reps, prof);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long hp[64];
  cudaMemcpy(hp, prof, sizeof(hp), cudaMemcpyDeviceToHost);
  const double per = ms * 1e3 / reps;
  const char* nm[9] = {"load", "l2_tail", "group_upd", "writeback", "trailing", "gram", "T", "l2_reduce", "l2_D"};
  printf("{\"panel\": \"%s\", \"nb\": %d, \"us_per_panel\": %.1f, \"phases_us\": {", name, NB, per);
  for (int i = 0; i < 9; ++i) printf("%s\"%s\": %.1f", i ? ", " : "", nm[i], hp[MODE * 16 + i] / 1e3 / reps);
  printf("}, \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
#ifdef TQR_PROF_L2
  unsigned long long l2[8];
  cudaMemcpyFromSymbol(l2, g_l2prof, sizeof(l2));
  const double cols = double(NB) * reps;
  printf("  level-2 cycles/column warp0: products+reduce %.0f  barrier %.0f  scalars %.0f  update %.0f | warp7: %.0f %.0f %.0f %.0f\n",
         l2[0] / cols, l2[1] / cols, l2[2] / cols, l2[3] / cols, l2[4] / cols, l2[5] / cols, l2[6] / cols, l2[7] / cols);
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(g_l2prof, z, sizeof(z));
#endif
  cudaFree(tiles);
  cudaFree(ts);
  cudaFree(prof);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<256, GE>("GEQRT", sms);
  run<256, TT>("TTQRT", sms);
  run<256, TS>("TSQRT", sms);
  run<64, GE>("GEQRT", sms);
  run<64, TT>("TTQRT", sms);
  return 0;
}
