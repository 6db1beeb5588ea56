// Dependent-chain latencies (cycles) of the FP64 ops on the panels' level-2
// critical path: DFMA, DADD, MUFU.RSQ64H / RCP64H (+ Newton), IEEE sqrt and
// division, SHFL, warp vote — one warp, clock64 around 256-long chains.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsq(double s) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s)); return y; }
__device__ __forceinline__ double rcp(double s) { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s)); return y; }

__global__ void lat(double* out, long long* cyc, double seed) {
  const int N = 256;
  double x = seed + threadIdx.x * 1e-9;
  long long t0, t1;
  int k = 0;
#define CHAIN(EXPR)                                   \
  t0 = clock64();                                     \
  for (int i = 0; i < N; ++i) { EXPR; }               \
  t1 = clock64();                                     \
  if (threadIdx.x == 0) cyc[k] = (t1 - t0) / N;       \
  ++k;
  CHAIN(x = fma(x, 0.999999, 1e-7))
  CHAIN(x = x + 1e-9)
  CHAIN(x = x * 1.0000001)
  CHAIN(x = rsq(x) + 1.0)
  CHAIN(x = rcp(x) + 1.0)
  CHAIN(x = sqrt(x) + 1.0)
  CHAIN(x = 1.0 / x + 1.0)
  CHAIN(x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9)
  CHAIN(x = __any_sync(0xffffffffu, x > 1e300) ? x : x + 1e-9)
  out[threadIdx.x] = x;
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 16 * 8);
  lat<<<1, 32>>>(o, c, 1.5);
  lat<<<1, 32>>>(o, c, 1.5);
  long long h[16];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[] = {"dfma", "dadd", "dmul", "rsqrt.approx.f64+dadd", "rcp.approx.f64+dadd", "sqrt(IEEE)+dadd",
                      "div(IEEE)+dadd", "shfl+dadd", "vote+sel+dadd"};
  printf("{");
  for (int i = 0; i < 9; ++i) printf("%s\"%s\": %lld", i ? ", " : "", nm[i], h[i]);
  printf("}\n");
  return 0;
}
