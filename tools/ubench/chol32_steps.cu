// Per-step clock64 trace of the warp-level 32x32 LDL^T + inverse sweep (potrf.cu design study).
// mode 0: shuffles, 1: smem LDS.128 broadcast, 2: smem without the inverse
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kLd = 65;
template <int kMode>
__global__ void k(const double* W, double* out, long long* t) {
  __shared__ double A[32 * kLd];
  __shared__ __align__(16) double cbuf[2][32];
  const int lane = threadIdx.x;
  for (int c = 0; c < 32; ++c) A[lane * kLd + c] = W[lane * 64 + c];
  __syncwarp();
  double a[32], sx[32], dd[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    a[c] = (c <= lane) ? A[lane * kLd + c] : 0.0;
    sx[c] = (c == lane) ? 1.0 : 0.0;
  }
  long long c0 = clock64();
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    double d;
    double* cb = cbuf[j & 1];
    if (kMode == 0) {
      d = __shfl_sync(0xffffffffu, a[j], j);
    } else {
      cb[lane] = a[j];
      __syncwarp();
      d = cb[j];
    }
    const double dinv = __drcp_rn(d);
    dd[j] = d;
    const double tt = a[j] * dinv;
    const double y = sx[j] * dinv;
    if (kMode == 0) {
#pragma unroll
      for (int c = j + 1; c < 32; ++c) {
        const double lc = __shfl_sync(0xffffffffu, a[j], c);
        a[c] = fma(-tt, lc, a[c]);
        sx[c] = fma(-lc, y, sx[c]);
      }
    } else {
#pragma unroll
      for (int c = (j + 1) & ~1; c < 32; c += 2) {
        const double2 lc = *reinterpret_cast<const double2*>(cb + c);
        if (c > j) {
          a[c] = fma(-tt, lc.x, a[c]);
          if (kMode == 1) sx[c] = fma(-lc.x, y, sx[c]);
        }
        a[c + 1] = fma(-tt, lc.y, a[c + 1]);
        if (kMode == 1) sx[c + 1] = fma(-lc.y, y, sx[c + 1]);
      }
    }
    if (lane == 0 && (j % 4 == 3)) t[j / 4] = clock64() - c0;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 32; ++c) s += a[c] + sx[c] + dd[c];
  out[lane] = s;
}
int main() {
  double h[64 * 64];
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) h[i * 64 + j] = (i == j ? 64.0 : 0.0) + 1.0 / (1 + i + j);
  double *d, *o; cudaMalloc(&d, sizeof h); cudaMalloc(&o, 256); cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  long long* t; cudaMalloc(&t, 8 * 8);
  long long ht[8];
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 32>>>(d, o, t); cudaMemcpy(ht, t, 64, cudaMemcpyDeviceToHost);
    printf("shfl      : "); for (int i = 0; i < 8; ++i) printf("%lld ", ht[i]); printf("\n");
    k<1><<<1, 32>>>(d, o, t); cudaMemcpy(ht, t, 64, cudaMemcpyDeviceToHost);
    printf("smem      : "); for (int i = 0; i < 8; ++i) printf("%lld ", ht[i]); printf("\n");
    k<2><<<1, 32>>>(d, o, t); cudaMemcpy(ht, t, 64, cudaMemcpyDeviceToHost);
    printf("smem noinv: "); for (int i = 0; i < 8; ++i) printf("%lld ", ht[i]); printf("\n");
  }
  return 0;
}
