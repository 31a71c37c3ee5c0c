// Timeline of the persistent potrf + TRSV kernel (CTA 0, %globaltimer) at n = 1024: per block step
// the time CTA 0 spends on its tiles (tile 0 = next diagonal block + its factorisation, the critical
// path) and waiting in the grid barrier, then the forward/backward TRSV barriers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Iinclude \
//        -o potrf_trace tools/ubench/potrf_trace.cu paper_2310_17556_b200/csrc/syrk_dmma.cu \
//        paper_2310_17556_b200/csrc/trsv.cu
// Round-2 final build, n = 1024: 16.4 us per block step (panel loads 1.6, two 64^3 DMMA GEMMs
// 4.5, chol_inv64 8.2, L / Linv stores 1.7), grid barrier ~1.1 us, backward solve 48 us.
#define FS_POTRF_TRACE 1
#include "../../paper_2310_17556_b200/csrc/potrf.cu"
#include <cstdio>
#include <vector>
#include <cmath>
using namespace fs;
int main() {
  const int64_t n = 1024;
  std::vector<double> h(n * n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) h[i * n + j] = (i == j ? (double)n : 0.0) + 1.0 / (1 + i + j);
  double *W, *W0, *scratch, *u, *z;
  int64_t* st;
  cudaMalloc(&W, n * n * 8); cudaMalloc(&W0, n * n * 8);
  cudaMalloc(&scratch, (size_t)(n * n + 4 * n * 64 + 8 * n + 64) * 8);
  cudaMalloc(&u, n * 8); cudaMalloc(&z, n * 8); cudaMalloc(&st, 8);
  cudaMemcpy(W0, h.data(), n * n * 8, cudaMemcpyHostToDevice);
  std::vector<double> hu(n, 1.0);
  cudaMemcpy(u, hu.data(), n * 8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(W, W0, n * n * 8, cudaMemcpyDeviceToDevice);
    cudaMemset(st, 0, 8);
    bool solved = false;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = potrf_lower(W, n, n, st, scratch, 0, nullptr, u, z, &solved);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long t[128];
    cudaMemcpyFromSymbol(t, g_potrf_trace, sizeof t);
    printf("rep %d: %.3f ms (%s, solved %d)\n", rep, ms, cudaGetErrorString(e), (int)solved);
    if (rep == 2) {
      printf("  diag0 factor %.1f us, barrier %.1f us\n", (t[1] - t[0]) / 1e3, (t[2] - t[1]) / 1e3);
      double work = 0, wait = 0;
      for (int k = 0; k < 15; ++k) {
        const double w = (t[3 + 2 * k] - (k ? t[2 + 2 * k] : t[2])) / 1e3, b2 = (t[4 + 2 * k] - t[3 + 2 * k]) / 1e3;
        work += w; wait += b2;
        printf("  step %2d: CTA0 tiles %.1f us, barrier %.1f us\n", k, w, b2);
      }
      printf("  steps total: tiles %.1f us, barriers %.1f us\n", work, wait);
      printf("  tail copy + last fwd block %.1f us, barrier %.1f us, backward solve %.1f us\n", (t[71] - t[70]) / 1e3,
             (t[72] - t[71]) / 1e3, (t[73] - t[72]) / 1e3);
      printf("  total (CTA 0) %.1f us\n", (t[73] - t[0]) / 1e3);
      const char* nm[] = {"A + old loads", "GEMM X = A Linv^T", "X -> smem", "GEMM X X^T + diag -> smem",
                          "(call)", "identity pad", "chol_inv64", "L/Linv store", "P copy"};
      const int a0[] = {80, 81, 82, 83, 84, 85, 86, 87, 88}, a1[] = {81, 82, 83, 84, 85, 86, 87, 88, 89};
      for (int i = 0; i < 9; ++i) printf("  step 5 critical: %-30s %.2f us\n", nm[i], (t[a1[i]] - t[a0[i]]) / 1e3);
    }
  }
  return 0;
}
