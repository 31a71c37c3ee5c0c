// H2D bandwidth: contiguous pinned copy vs 2-D column-block copies (n rows x m/C cols).
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t n = 1024, m = 1000000, elem = 4;
  void *h, *d;
  cudaMallocHost(&h, n * m * elem);
  cudaMalloc(&d, n * m * elem);
  memset(h, 0, n * m * elem);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, st);
    cudaMemcpyAsync(d, h, n * m * elem, cudaMemcpyHostToDevice, st);
    cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("contiguous: %.2f ms %.1f GB/s\n", ms, n * m * elem / ms / 1e6);
  }
  int Cs[] = {1, 2, 4, 8, 16, 32, 64};
  for (int C : Cs) {
    const size_t w = (m + C - 1) / C;
    cudaEventRecord(a, st);
    for (int c = 0; c < C; ++c) {
      const size_t c0 = c * w, cw = (c0 + w > m ? m - c0 : w);
      cudaMemcpy2DAsync((char*)d + c0 * elem, m * elem, (char*)h + c0 * elem, m * elem, cw * elem, n,
                        cudaMemcpyHostToDevice, st);
    }
    cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("2-D column blocks C=%d (%zu KB segments): %.2f ms %.1f GB/s\n", C, w * elem / 1024, ms,
           n * m * elem / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
