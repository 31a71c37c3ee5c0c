// complex.cu — complex score matrices reduced to the real path.
//
// solve_realpart (solvers.py:216-240): C = [Re S; Im S] (2n x m, sr.py:61-70), C^T C = Re[S^H S].
// solve_chol_hermitian (solvers.py:209-213): the real representation
//   rho(S) = [[Re S, -Im S], [Im S, Re S]] (2n x 2m)  with  rho(S)^T rho(S) = rho(S^H S),
// so (S^H S + lam I) x = v  <=>  (rho^T rho + lam I) [Re x; Im x] = [Re v; Im v], solved by the
// plain real route (tensor-core Gram of the 2n rows, fp64 potrf, ...).  One streaming pass
// de-interleaves the (re, im) pairs into the aligned real layout.
#include "common.cuh"
#include "kernels.h"

namespace fs {
namespace {

template <typename T>
__global__ void embed_kernel(const T* __restrict__ S, int64_t n, int64_t m, int64_t ldS, int kind, T* __restrict__ out,
                             int64_t ldo) {
  // grid-stride over (row i < n, column j < m); S holds (re, im) pairs, ldS in complex elements
  const int64_t total = n * m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / m, j = e - i * m;
    const T re = S[2 * (i * ldS + j)], im = S[2 * (i * ldS + j) + 1];
    if (kind == 0) {
      out[i * ldo + j] = re;
      out[(n + i) * ldo + j] = im;
    } else {
      out[i * ldo + j] = re;
      out[i * ldo + m + j] = -im;
      out[(n + i) * ldo + j] = im;
      out[(n + i) * ldo + m + j] = re;
    }
  }
}

}  // namespace

cudaError_t embed_complex(bool f64, const void* S, int64_t n, int64_t m, int64_t ldS, int kind, void* out, int64_t ldo,
                          int num_sms, cudaStream_t st, int* launches) {
  const unsigned grid = (unsigned)(num_sms * 8);
  if (f64) embed_kernel<double><<<grid, 256, 0, st>>>((const double*)S, n, m, ldS, kind, (double*)out, ldo);
  else embed_kernel<float><<<grid, 256, 0, st>>>((const float*)S, n, m, ldS, kind, (float*)out, ldo);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace fs
