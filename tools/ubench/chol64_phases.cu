// Phase timing (clock64) of potrf.cu's chol_inv64 structure on one 64x64 tile.
#include "../../paper_2310_17556_b200/csrc/potrf.cu"
#include <cstdio>
using namespace fs;
__device__ int chol_inv64_t(double (*A)[kLd], double (*X)[kLd], double (*T)[kLd], long long* ts) {
  __shared__ int sfail;
  __shared__ __align__(16) double colbuf[2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  if (warp == 0) {
    const int f = warp_chol_inv32(&A[0][0], &X[0][0], colbuf);
    if (lane == 0) sfail = f;
  } else if (warp == 1) {
    for (int c = 0; c < 32; ++c) X[lane][32 + c] = 0.0;
  }
  __syncthreads();
  long long t1 = clock64();
  if (sfail >= 0) return sfail;
  double acc[2][2];
  gemm32_dmma<true>(&A[32][0], &X[0][0], acc);
  __syncthreads();
  store32_dmma(&A[32][0], acc, 1.0, false);
  __syncthreads();
  long long t2 = clock64();
  gemm32_dmma<true>(&A[32][0], &A[32][0], acc);
  store32_dmma(&A[32][32], acc, -1.0, true);
  __syncthreads();
  long long t3 = clock64();
  if (warp == 0) {
    const int f = warp_chol_inv32(&A[32][32], &X[32][32], colbuf);
    if (lane == 0) sfail = f < 0 ? -1 : 32 + f;
  }
  __syncthreads();
  long long t4 = clock64();
  if (sfail >= 0) return sfail;
  gemm32_dmma<false>(&A[32][0], &X[0][0], acc);
  store32_dmma(&T[0][0], acc, 1.0, false);
  __syncthreads();
  gemm32_dmma<false>(&X[32][32], &T[0][0], acc);
  store32_dmma(&X[32][0], acc, -1.0, false);
  __syncthreads();
  long long t5 = clock64();
  if (threadIdx.x == 0) { ts[0] = t1 - t0; ts[1] = t2 - t1; ts[2] = t3 - t2; ts[3] = t4 - t3; ts[4] = t5 - t4; }
  return -1;
}
__global__ void __launch_bounds__(256) k(const double* W, long long* t) {
  extern __shared__ double dsm[];
  double (*A)[65] = reinterpret_cast<double (*)[65]>(dsm);
  double (*X)[65] = reinterpret_cast<double (*)[65]>(dsm + 64 * 65);
  double (*B)[65] = reinterpret_cast<double (*)[65]>(dsm + 2 * 64 * 65);
  for (int rep = 0; rep < 3; ++rep) {
    load_tile(W, 64, 64, 0, 0, A);
    __syncthreads();
    chol_inv64_t(A, X, B, t + rep * 5);
  }
}
int main() {
  double h[64 * 64];
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) h[i * 64 + j] = (i == j ? 64.0 : 0.0) + 1.0 / (1 + i + j);
  double* d; cudaMalloc(&d, sizeof h); cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  long long* t; cudaMalloc(&t, 15 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 64 * 65 * 8);
  k<<<1, 256, 3 * 64 * 65 * 8>>>(d, t);
  long long ht[15]; cudaMemcpy(ht, t, sizeof ht, cudaMemcpyDeviceToHost);
  for (int r = 0; r < 3; ++r)
    printf("chol32a %lld  L10 %lld  A11upd %lld  chol32b %lld  X10 %lld\n", ht[r * 5], ht[r * 5 + 1], ht[r * 5 + 2],
           ht[r * 5 + 3], ht[r * 5 + 4]);
  return 0;
}
