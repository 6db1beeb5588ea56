// cudaMemcpy2DAsync H2D rate for column blocks of a pinned row-major
// 16384 x 16384 fp64 matrix, by block width (tiles of 256 columns).
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const long long m = 16384, n = 16384;
  double *h, *d;
  cudaHostAlloc(&h, m * n * 8, cudaHostAllocDefault);
  for (long long x = 0; x < m * n; x += 512) h[x] = 1.0;
  cudaMalloc(&d, m * n * 8);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int ws[] = {64, 1, 2, 4, 8, 16};
  for (int w : ws) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0, s);
      if (w == 64) {
        for (int r = 0; r < 64; ++r)
          cudaMemcpyAsync(d + r * 256 * n, h + r * 256 * n, 256 * n * 8, cudaMemcpyHostToDevice, s);
      } else {
        for (int j = 0; j < 64 / w; ++j)
          cudaMemcpy2DAsync(d + j * 256 * w, n * 8, h + j * 256 * w, n * 8, 256 * w * 8, m, cudaMemcpyHostToDevice, s);
      }
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("width %2d tiles (%6d B segments): %.2f ms  %.1f GB/s\n", w, 2048 * w, ms, m * n * 8 / 1e6 / ms);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
