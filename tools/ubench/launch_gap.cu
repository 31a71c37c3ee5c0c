// Launch-to-launch cost of the solve's kernel shapes when chained on one stream (each kernel
// trivially short): plain 148-CTA grid, 132 CTAs in 4-CTA clusters with ~225 KB of shared memory
// (the x + y pass's shape), one 16-CTA non-portable cluster (the TRSV pair's shape), and a
// cooperative 148-CTA launch (potrf's).  Prints microseconds per launch.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_plain(int* p) { if (threadIdx.x == 0 && p) p[blockIdx.x] = 1; }
__global__ void __cluster_dims__(4, 1, 1) k_cl4(int* p) { if (threadIdx.x == 0 && p) p[blockIdx.x] = 1; }
__global__ void k_cl16(int* p) { if (threadIdx.x == 0 && p) p[blockIdx.x] = 1; }

int main() {
  int* d;
  cudaMalloc(&d, 4096 * 4);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int N = 200;
  auto timeit = [&](const char* name, auto launch) {
    for (int i = 0; i < 10; ++i) launch();
    cudaStreamSynchronize(st);
    cudaEventRecord(a, st);
    for (int i = 0; i < N; ++i) launch();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %.2f us per launch (%s)\n", name, ms * 1e3 / N, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("plain 148 x 512", [&] { k_plain<<<148, 512, 0, st>>>(d); });
  cudaFuncSetAttribute(k_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  timeit("plain 148 x 512, 225 KB smem", [&] { k_plain<<<148, 512, 225 * 1024, st>>>(d); });
  cudaFuncSetAttribute(k_cl4, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  timeit("4-CTA clusters x 33, 512 thr, 225 KB", [&] { k_cl4<<<132, 512, 225 * 1024, st>>>(d); });
  cudaFuncSetAttribute(k_cl16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_cl16, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  timeit("one 16-CTA cluster, 256 thr, 150 KB", [&] {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 150 * 1024;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_cl16, d);
  });
  timeit("cooperative 148 x 256", [&] {
    void* args[] = {&d};
    cudaLaunchCooperativeKernel((const void*)k_plain, dim3(148), dim3(256), args, 0, st);
  });
  timeit("1 CTA x 1024", [&] { k_plain<<<1, 1024, 0, st>>>(d); });
  return 0;
}
