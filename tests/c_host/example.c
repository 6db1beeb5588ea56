/* A plain C host of the C ABI (include/tqr.h) — what a non-Python binding of
 * the reference's QR path would do.  Schedule part runs
 * without a GPU; with "gpu" it factors a seeded 1024 x 512 fp64 matrix
 * (nb = 64, Greedy/TT) on the device and checks ||R||_F = ||A||_F and R's
 * triangularity.  Built and run by tests/test_cli_abi.py (CPU part) and
 * tests/test_numeric_gpu.py (GPU part). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "tqr.h"

/* minimal CUDA runtime prototypes (libcudart) so the example needs no CUDA headers */
typedef int cudaError_t;
extern cudaError_t cudaMalloc(void** p, size_t n);
extern cudaError_t cudaFree(void* p);
extern cudaError_t cudaMemcpy(void* d, const void* s, size_t n, int kind);
extern cudaError_t cudaMemset(void* d, int v, size_t n);
extern cudaError_t cudaDeviceSynchronize(void);
#define H2D 1
#define D2H 2

static int fail(const char* what) {
  fprintf(stderr, "FAIL %s: %s\n", what, tqr_last_error());
  return 1;
}

int main(int argc, char** argv) {
  tqr_build* b = NULL;
  tqr_build_info info;
  if (tqr_build_tree(8, 4, "greedy", 0, TQR_NO_BS, 1, NULL, 1, 0, &b) != TQR_OK) return fail("build_tree");
  if (tqr_build_get_info(b, &info) != TQR_OK) return fail("get_info");
  printf("greedy 8x4: cp %lld, total weight %lld\n", (long long)info.cp, (long long)info.total_weight);
  if (info.cp != 78 || info.total_weight != 640) return fail("golden cp / weight");
  tqr_build_free(b);
  /* errors carry the reference's messages */
  if (tqr_build_tree(3, 5, "greedy", 0, TQR_NO_BS, 1, NULL, 1, 0, &b) != TQR_EVALUE) return fail("p < q accepted");
  printf("p < q rejected: %s\n", tqr_last_error());
  if (argc < 2 || strcmp(argv[1], "gpu") != 0) {
    printf("schedule ok\n");
    return 0;
  }

  const int p = 16, q = 8, nb = 64;
  const int64_t m = (int64_t)p * nb, n = (int64_t)q * nb;
  tqr_plan* plan = NULL;
  tqr_plan_info pi;
  if (tqr_build_tree(p, q, "greedy", 0, TQR_NO_BS, 1, NULL, 1, 0, &b) != TQR_OK) return fail("build_tree");
  if (tqr_plan_create(b, 100, 32, &plan) != TQR_EVALUE) return fail("nb = 100 accepted");
  printf("nb = 100 rejected: %s\n", tqr_last_error());
  if (tqr_plan_create(b, nb, 32, &plan) != TQR_OK) return fail("plan_create");
  if (tqr_plan_get_info(plan, &pi) != TQR_OK) return fail("plan_info");

  double* A = malloc(sizeof(double) * m * n);
  double* R = malloc(sizeof(double) * n * n);
  unsigned long long s = 12345;
  double na2 = 0.0;
  for (int64_t e = 0; e < m * n; ++e) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    A[e] = (double)((s >> 11) & 0xfffff) / (double)0xfffff - 0.5;
    na2 += A[e] * A[e];
  }
  double *dA, *dT, *dTG, *dTE, *dR;
  if (cudaMalloc((void**)&dA, sizeof(double) * m * n) || cudaMalloc((void**)&dT, sizeof(double) * m * n) ||
      cudaMalloc((void**)&dTG, sizeof(double) * p * q * pi.tg_stride) ||
      cudaMalloc((void**)&dTE, sizeof(double) * p * q * pi.te_stride) || cudaMalloc((void**)&dR, sizeof(double) * n * n))
    return fail("cudaMalloc");
  cudaMemset(dTG, 0, sizeof(double) * p * q * pi.tg_stride);
  cudaMemset(dTE, 0, sizeof(double) * p * q * pi.te_stride);
  cudaMemcpy(dA, A, sizeof(double) * m * n, H2D);
  int rc = tqr_pack(dA, n, 1, dT, p, q, nb, NULL);
  if (rc == TQR_OK) rc = tqr_factor(plan, dT, dTG, dTE, NULL);
  if (rc == TQR_OK) rc = tqr_extract_r(dT, p, q, nb, dR, n, 1, NULL);
  if (rc != TQR_OK) return fail("pack/factor/extract");
  cudaDeviceSynchronize();
  cudaMemcpy(R, dR, sizeof(double) * n * n, D2H);
  double nr2 = 0.0, below = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const double v = R[i * n + j];
      if (j >= i) nr2 += v * v; else below += fabs(v);
    }
  const double rel = fabs(sqrt(nr2) - sqrt(na2)) / sqrt(na2);
  printf("||R||_F vs ||A||_F rel diff %.3e, |R below diag| %.1e, items %lld\n", rel, below, (long long)pi.n_items);
  cudaFree(dA); cudaFree(dT); cudaFree(dTG); cudaFree(dTE); cudaFree(dR);
  free(A); free(R);
  tqr_plan_free(plan);
  tqr_build_free(b);
  if (!(rel < 1e-13) || below != 0.0) return fail("numerics");
  printf("gpu ok\n");
  return 0;
}
