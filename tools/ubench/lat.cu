// Dependent-chain latencies on sm_100a: DFMA, DADD, fp64 div, rcp, LDS.64, SHFL(double), FFMA.
#include <cstdio>
__global__ void lat_kernel(double* out, long long* t, double a, double b) {
  __shared__ double sm[256];
  sm[threadIdx.x] = threadIdx.x * 1.0;
  __syncthreads();
  double x = a; long long c0, c1;
  c0 = clock64(); for (int i = 0; i < 1000; ++i) x = fma(x, b, a); c1 = clock64(); t[0] = c1 - c0;
  c0 = clock64(); for (int i = 0; i < 1000; ++i) x = x + b; c1 = clock64(); t[1] = c1 - c0;
  c0 = clock64(); for (int i = 0; i < 100; ++i) x = a / x; c1 = clock64(); t[2] = (c1 - c0) * 10;
  c0 = clock64(); for (int i = 0; i < 1000; ++i) x = __drcp_rn(x); c1 = clock64(); t[3] = c1 - c0;
  int idx = 0;
  c0 = clock64(); for (int i = 0; i < 1000; ++i) { double v = sm[idx]; idx = ((int)v + 1) & 255; x += v; } c1 = clock64(); t[4] = c1 - c0;
  c0 = clock64(); for (int i = 0; i < 1000; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0; c1 = clock64(); t[5] = c1 - c0;
  float y = (float)a;
  c0 = clock64(); for (int i = 0; i < 1000; ++i) y = fmaf(y, (float)b, (float)a); c1 = clock64(); t[6] = c1 - c0;
  c0 = clock64(); for (int i = 0; i < 100; ++i) x = sqrt(x + 1.0); c1 = clock64(); t[7] = (c1 - c0) * 10;
  out[threadIdx.x] = x + y;
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 256 * 8); cudaMalloc(&t, 8 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    lat_kernel<<<1, 32>>>(o, t, 1.0000001, 0.9999999);
    long long h[8]; cudaMemcpy(h, t, 64, cudaMemcpyDeviceToHost);
    printf("per-op cycles: DFMA %.1f DADD %.1f DDIV %.1f DRCP %.1f LDS64 %.1f SHFL64+DADD %.1f FFMA %.1f DSQRT %.1f\n",
           h[0] / 1e3, h[1] / 1e3, h[2] / 1e3, h[3] / 1e3, h[4] / 1e3, h[5] / 1e3, h[6] / 1e3, h[7] / 1e3);
  }
  return 0;
}
