// Verification kernel for dmath.cuh: evaluates the library function and its
// constant-bank restatement on the same inputs so a test can require equal
// bits (cdvz_gpu_math_check). Not on the extraction path.
#include "common.cuh"
#include "dmath.cuh"

namespace cdvz_gpu {

namespace {
__global__ void k_math_check(int fn, const double* a, const double* b, long long n, double* lib, double* ours) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (fn == 0) {
      lib[i] = ::atan2(a[i], b[i]);
      ours[i] = dm::atan2(a[i], b[i]);
    } else {
      lib[i] = ::exp(a[i]);
      ours[i] = dm::exp(a[i]);
    }
  }
}
}  // namespace

cudaError_t launch_math_check(int fn, const double* a, const double* b, long long n, double* lib, double* ours,
                              cudaStream_t st) {
  k_math_check<<<148 * 8, 256, 0, st>>>(fn, a, b, n, lib, ours);
  return cudaGetLastError();
}

}  // namespace cdvz_gpu
