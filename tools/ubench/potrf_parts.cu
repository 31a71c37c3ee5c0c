// Microbenchmark: clock64 timing of potrf.cu's device building blocks on one 64x64 tile.
#include "../../paper_2310_17556_b200/csrc/potrf.cu"
#include <cstdio>
using namespace fs;
__global__ void __launch_bounds__(256) parts_kernel(const double* W, long long* t) {
  extern __shared__ double dsm[];
  double (*A)[65] = reinterpret_cast<double (*)[65]>(dsm);
  double (*X)[65] = reinterpret_cast<double (*)[65]>(dsm + 64 * 65);
  double (*B)[65] = reinterpret_cast<double (*)[65]>(dsm + 2 * 64 * 65);
  __shared__ double rd[64];
  __shared__ int fail;
  long long c0 = clock64();
  load_tile(W, 64, 64, 0, 0, A);
  __syncthreads();
  long long c1 = clock64();
  factor_block(A, 64, &fail);
  __syncthreads();
  long long c2 = clock64();
  if (threadIdx.x < 64) rd[threadIdx.x] = 1.0 / A[threadIdx.x][threadIdx.x];
  for (int e = threadIdx.x; e < 64 * 64; e += 256) X[e / 64][e % 64] = W[e] * 0.5;
  __syncthreads();
  long long c3 = clock64();
  trsm_rows(A, rd, X);
  __syncthreads();
  long long c4 = clock64();
  double acc[4][4];
  gemm_nt(X, A, acc);
  __syncthreads();
  long long c5 = clock64();
  if (threadIdx.x == 0) { t[0] = c1 - c0; t[1] = c2 - c1; t[2] = c4 - c3; t[3] = c5 - c4; t[4] = (long long)acc[0][0]; }
}
int main() {
  double h[64 * 64];
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) h[i * 64 + j] = (i == j ? 64.0 : 0.0) + 1.0 / (1 + i + j);
  double* d; cudaMalloc(&d, sizeof h); cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  long long* t; cudaMalloc(&t, 64);
  cudaFuncSetAttribute(parts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 64 * 65 * 8);
  for (int rep = 0; rep < 3; ++rep) {
    parts_kernel<<<1, 256, 3 * 64 * 65 * 8>>>(d, t);
    long long ht[5]; cudaMemcpy(ht, t, 40, cudaMemcpyDeviceToHost);
    printf("cycles: load %lld  factor %lld  trsm %lld  gemm %lld   (%s)\n", ht[0], ht[1], ht[2], ht[3], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
