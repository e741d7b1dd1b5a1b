// sad_precond.cu -- instantiation and dispatch of the triangular-solve kernel
// (sad_precond.cuh): block type (fp64 / complex128) x factor value type x R.
#include <cuda_runtime.h>

#include "sad_precond.cuh"

namespace sad {

void count_launches(long long k);   // sad_capi.cu

template <typename XT, typename VT>
static int sptrsv_r(const TriArgs& a, int R, int grid, cudaStream_t s) {
  switch (R) {
    case 1: k_sptrsv<XT, VT, 1><<<grid, kThreads, 0, s>>>(a); break;
    case 2: k_sptrsv<XT, VT, 2><<<grid, kThreads, 0, s>>>(a); break;
    case 3: k_sptrsv<XT, VT, 3><<<grid, kThreads, 0, s>>>(a); break;
    case 4: k_sptrsv<XT, VT, 4><<<grid, kThreads, 0, s>>>(a); break;
    case 5: k_sptrsv<XT, VT, 5><<<grid, kThreads, 0, s>>>(a); break;
    case 6: k_sptrsv<XT, VT, 6><<<grid, kThreads, 0, s>>>(a); break;
    case 7: k_sptrsv<XT, VT, 7><<<grid, kThreads, 0, s>>>(a); break;
    case 8: k_sptrsv<XT, VT, 8><<<grid, kThreads, 0, s>>>(a); break;
    default: return 1;
  }
  count_launches(1);
  return 0;
}

// block_complex: the n x R block is complex128; vals_complex: the factor is.
// A complex factor needs a complex block.
int sptrsv_launch(const TriArgs& a, int R, bool block_complex, bool vals_complex, int grid,
                  cudaStream_t s) {
  if (!block_complex) {
    if (vals_complex) return 1;
    return sptrsv_r<double, double>(a, R, grid, s);
  }
  return vals_complex ? sptrsv_r<double2, double2>(a, R, grid, s)
                      : sptrsv_r<double2, double>(a, R, grid, s);
}

}  // namespace sad
