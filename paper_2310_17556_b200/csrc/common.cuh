// common.cuh — shared device helpers for the fisher-b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define FS_DEVINL __device__ __forceinline__

namespace fs {

constexpr int kWarp = 32;

template <typename T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<double> { using type = double4; };  // 32-byte vector (sm_100 LDG.256)

FS_DEVINL double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// N independent warp sums, interleaved: five rounds of N independent shuffles instead of N
// dependent five-shuffle chains (the same xor order per value: bit-identical to warp_sum).  On
// the TRSV's critical path 8 chained sums cost ~1 us per block.
template <int N>
FS_DEVINL void warp_sum_n(double (&v)[N]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
}

// Streaming (read-once) loads: keep S out of L1, (L2 evict hints need 256-bit vectors).
FS_DEVINL float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
FS_DEVINL double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
FS_DEVINL float ld_stream(const float* p) { return __ldg(p); }
FS_DEVINL double ld_stream(const double* p) { return __ldg(p); }

template <typename T> FS_DEVINL double to_d(T x) { return static_cast<double>(x); }

}  // namespace fs
