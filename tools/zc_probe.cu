// Zero-copy read probe: CTAs transpose 256x256 tiles straight out of pinned,
// row-major host memory (the PACK pattern) into device tiles.  Reports the
// aggregate PCIe read rate for several grid sizes and the single-CTA rate.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NB = 256, NT = 256, CR = 32, LD = NB + 1, PER = CR * NB / NT;
__global__ void __launch_bounds__(NT, 1) zc_pack(const double* __restrict__ a, long long lda, double* tiles, int p,
                                                 int q, int ntiles) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int i = t % p, j = t / p;  // tile-column-major order
    const double* src = a + (long long)i * NB * lda + (long long)j * NB;
    double* dst = tiles + (size_t(j) * p + i) * NB * NB;
    double v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * NT;
      v[u] = __ldcv(src + (long long)(e / NB) * lda + e % NB);
    }
    for (int r0 = 0; r0 < NB; r0 += CR) {
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int e = tid + u * NT;
        sm[(e / NB) * LD + e % NB] = v[u];
      }
      __syncthreads();
      if (r0 + CR < NB) {
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int e = tid + u * NT;
          v[u] = __ldcv(src + (long long)(r0 + CR + e / NB) * lda + e % NB);
        }
      }
      for (int c = warp; c < NB; c += NT / 32) __stcg(dst + size_t(c) * NB + r0 + lane, sm[lane * LD + c]);
      __syncthreads();
    }
  }
}
int main() {
  const int p = 64, q = 64;
  const long long m = p * NB, n = q * NB;
  double* h;
  cudaHostAlloc(&h, m * n * 8, cudaHostAllocDefault);
  for (long long x = 0; x < m * n; ++x) h[x] = double(x % 1000);
  double* d;
  cudaMalloc(&d, m * n * 8);
  const size_t smem = CR * LD * 8;
  cudaFuncSetAttribute(zc_pack, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int grids[] = {1, 8, 32, 64, 148, 296};
  for (int g : grids) {
    const int nt = g == 1 ? 16 : (g < 148 ? 4 * g : p * q);
    zc_pack<<<g, NT, smem>>>(h, n, d, p, q, nt);
    cudaEventRecord(e0);
    zc_pack<<<g, NT, smem>>>(h, n, d, p, q, nt);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gb = double(nt) * NB * NB * 8 / 1e9;
    printf("grid %4d tiles %5d: %.3f ms  %.1f GB/s  per-CTA %.2f GB/s  per-tile %.1f us\n", g, nt, ms, gb / (ms * 1e-3),
           gb / (ms * 1e-3) / g, ms * 1e3 / (double(nt) / g));
  }
  // check
  double* t = (double*)malloc(NB * NB * 8);
  cudaMemcpy(t, d + (size_t(3) * p + 5) * NB * NB, NB * NB * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < NB; ++r)
    for (int c = 0; c < NB; ++c)
      if (t[r + c * NB] != h[(5LL * NB + r) * n + 3 * NB + c]) ++bad;
  printf("check bad=%d err=%s\n", bad, cudaGetErrorString(cudaGetLastError()));
}
