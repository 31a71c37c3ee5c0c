// Microbenchmark: clock64 timing of potrf.cu's device building blocks on one 64x64 tile.
#include "../../paper_2310_17556_b200/csrc/potrf.cu"
#include <cstdio>
using namespace fs;
__global__ void __launch_bounds__(256) parts_kernel(const double* W, long long* t, int reps) {
  extern __shared__ double dsm[];
  double (*A)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm);
  double (*X)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + 64 * kLd);
  double (*B)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + 2 * 64 * kLd);
  for (int rep = 0; rep < reps; ++rep) {
    long long c0 = clock64();
    load_tile(W, 64, 64, 0, 0, A);
    __syncthreads();
    long long c1 = clock64();
    int f = -1;
    __shared__ __align__(16) double cb0[2][32];
    if ((threadIdx.x >> 5) == 0) f = warp_chol_inv32(&A[0][0], &X[0][0], cb0);
    __syncthreads();
    long long c2 = clock64();
    load_tile(W, 64, 64, 0, 0, A);
    __syncthreads();
    long long c3 = clock64();
    f += chol_inv64(A, X, B);
    __syncthreads();
    long long c4 = clock64();
    double acc[4][4];
    gemm_nt(X, A, acc);
    __syncthreads();
    long long c5 = clock64();
    if (threadIdx.x == 0) {
      t[rep * 6 + 0] = c1 - c0; t[rep * 6 + 1] = c2 - c1; t[rep * 6 + 2] = c4 - c3; t[rep * 6 + 3] = c5 - c4;
      t[rep * 6 + 4] = (long long)acc[0][0] + f;
    }
  }
}
int main() {
  double h[64 * 64];
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) h[i * 64 + j] = (i == j ? 64.0 : 0.0) + 1.0 / (1 + i + j);
  double* d; cudaMalloc(&d, sizeof h); cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  long long* t; cudaMalloc(&t, 6 * 8 * 4);
  cudaFuncSetAttribute(parts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 64 * kLd * 8);
  for (int launch = 0; launch < 2; ++launch) {
    parts_kernel<<<1, 256, 3 * 64 * kLd * 8>>>(d, t, 3);
    long long ht[18]; cudaMemcpy(ht, t, sizeof ht, cudaMemcpyDeviceToHost);
    for (int rep = 0; rep < 3; ++rep)
      printf("launch %d rep %d cycles: load %lld  chol_inv32 %lld  chol_inv64 %lld  gemm_nt64 %lld  (%s)\n", launch, rep,
             ht[rep * 6], ht[rep * 6 + 1], ht[rep * 6 + 2], ht[rep * 6 + 3], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
