// FP64 peak probe for B200 (sm_100a): DMMA.8x8x4 (mma.sync f64) and DFMA loops,
// plus a fragment-layout self check.  Prints one JSON line.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters, double a0, double b0) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters, double a0, double b0) {
  double c[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i] = i;
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

// one warp: A 8x4 row-major, B 4x8, C 8x8 ; assumed layouts:
// a: row=lane>>2 col=lane&3 ; b: row(k)=lane&3 col(n)=lane>>2 ; c: row=lane>>2 col=2*(lane&3)+i
__global__ void k_layout(const double* A, const double* B, double* C) {
  int l = threadIdx.x;
  double a = A[(l >> 2) * 4 + (l & 3)];
  double b = B[(l & 3) * 8 + (l >> 2)];
  double c0 = 0, c1 = 0;
  dmma(c0, c1, a, b);
  C[(l >> 2) * 8 + 2 * (l & 3) + 0] = c0;
  C[(l >> 2) * 8 + 2 * (l & 3) + 1] = c1;
}

__global__ void k_lat(double* out, long long* cyc, int n) {
  double c0 = 0, c1 = 0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) dmma(c0, c1, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[1] = c0 + c1; }
}
// one warp per SMSP, k chains: cycles per DMMA issue
template <int CH>
__global__ void k_thr(double* out, long long* cyc, int n) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) dmma(c[k][0], c[k][1], a, b);
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < CH; ++i) s += c[i][0];
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[2] = s; }
}

int main(int argc, char** argv) {
  double* d; cudaMalloc(&d, 1024 * sizeof(double));
  // layout check
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = i + 1; hB[i] = 100 + 3 * i; }
  for (int m = 0; m < 8; ++m) for (int n = 0; n < 8; ++n) {
    double s = 0; for (int k = 0; k < 4; ++k) s += hA[m * 4 + k] * hB[k * 8 + n]; ref[m * 8 + n] = s; }
  cudaMemcpy(d, hA, 32 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d + 32, hB, 32 * 8, cudaMemcpyHostToDevice);
  k_layout<<<1, 32>>>(d, d + 32, d + 64);
  cudaMemcpy(hC, d + 64, 64 * 8, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < 64; ++i) bad += (hC[i] != ref[i]);
  int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  auto timeit = [&](auto launch, double flops_per_launch) {
    launch(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    return flops_per_launch / (best * 1e-3) / 1e12;
  };
  printf("{\"layout_ok\": %s, \"sms\": %d", bad ? "false" : "true", sms);
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * (wpb <= 8 ? 2 : 1);
    double fl = 2.0 * 256 * 8 * (double)iters * blocks * wpb;
    double t = timeit([&] { k_dmma<8><<<blocks, 32 * wpb>>>(d, iters, 1.0, 1.0); }, fl);
    printf(", \"dmma_w%d_tf\": %.2f", wpb, t);
  }
  {
    int blocks = sms * 2, wpb = 8;
    double fl = 2.0 * 256 * 4 * (double)iters * blocks * wpb;
    double t = timeit([&] { k_dmma<4><<<blocks, 32 * wpb>>>(d, iters, 1.0, 1.0); }, fl);
    printf(", \"dmma_ch4_w8x2_tf\": %.2f", t);
    fl = 2.0 * 256 * 2 * (double)iters * blocks * wpb;
    t = timeit([&] { k_dmma<2><<<blocks, 32 * wpb>>>(d, iters, 1.0, 1.0); }, fl);
    printf(", \"dmma_ch2_w8x2_tf\": %.2f", t);
    fl = 2.0 * 256 * 1 * (double)iters * blocks * wpb;
    t = timeit([&] { k_dmma<1><<<blocks, 32 * wpb>>>(d, iters, 1.0, 1.0); }, fl);
    printf(", \"dmma_ch1_w8x2_tf\": %.2f", t);
    fl = 2.0 * 256 * 8 * (double)iters * sms * 1;
    t = timeit([&] { k_dmma<8><<<sms, 32>>>(d, iters, 1.0, 1.0); }, fl);
    printf(", \"dmma_1warp_per_sm_tf\": %.2f", t);
    fl = 2.0 * 256 * 8 * (double)iters * sms * 4;
    t = timeit([&] { k_dmma<8><<<sms, 128>>>(d, iters, 1.0, 1.0); }, fl);
    printf(", \"dmma_4warp_per_sm_tf\": %.2f", t);
  }
  for (int wpb : {8, 16}) {
    int blocks = sms * 4;
    double fl = 2.0 * 32 * 8 * (double)iters * blocks * wpb;
    double t = timeit([&] { k_dfma<8><<<blocks, 32 * wpb>>>(d, iters, 1.0000001, 1e-7); }, fl);
    printf(", \"dfma_w%d_tf\": %.2f", wpb, t);
  }
  {
    long long* dc; cudaMalloc(&dc, 64); long long hc;
    k_lat<<<1, 32>>>(d, dc, 4096); cudaMemcpy(&hc, dc, 8, cudaMemcpyDeviceToHost);
    printf(", \"dmma_latency_cyc\": %.1f", hc / 4096.0);
    k_thr<2><<<1, 32>>>(d, dc, 2048); cudaMemcpy(&hc, dc, 8, cudaMemcpyDeviceToHost);
    printf(", \"dmma_cyc_per_issue_2ch\": %.2f", hc / 4096.0);
    k_thr<4><<<1, 32>>>(d, dc, 1024); cudaMemcpy(&hc, dc, 8, cudaMemcpyDeviceToHost);
    printf(", \"dmma_cyc_per_issue_4ch\": %.2f", hc / 4096.0);
    k_thr<8><<<1, 32>>>(d, dc, 512); cudaMemcpy(&hc, dc, 8, cudaMemcpyDeviceToHost);
    printf(", \"dmma_cyc_per_issue_8ch\": %.2f", hc / 4096.0);
    k_thr<8><<<1, 64>>>(d, dc, 512); cudaMemcpy(&hc, dc, 8, cudaMemcpyDeviceToHost);
    printf(", \"dmma_cyc_per_issue_8ch_2warps\": %.2f", hc / 4096.0);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
