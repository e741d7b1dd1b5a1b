// sad_minres.cu -- instantiation and dispatch of the MINRES kernels
// (sad_minres.cuh).  Compiled once per -DSAD_MINRES_PART=<0|1>: fp64 /
// complex128 blocks, so the two halves build in parallel.
#include <cuda_runtime.h>
#include <cstdio>

#include "sad_minres.cuh"

#ifndef SAD_MINRES_PART
#error "compile with -DSAD_MINRES_PART=<0|1>"
#endif

namespace sad {

void count_launches(long long k);   // sad_capi.cu

#if SAD_MINRES_PART == 0
using XT_ = double;
#else
using XT_ = double2;
#endif

template <int R>
static void vec_r(int K, const MArgs& a, int grid, cudaStream_t s) {
  switch (K) {
    case MR_START: k_mr_vec<XT_, R, MR_START><<<grid, kThreads, 0, s>>>(a); break;
    case MR_YUPD: k_mr_vec<XT_, R, MR_YUPD><<<grid, kThreads, 0, s>>>(a); break;
    case MR_WUPD: k_mr_vec<XT_, R, MR_WUPD><<<grid, kThreads, 0, s>>>(a); break;
  }
}

template <typename VT, int R, bool SIGMA>
static void spmm_k(int K, const MArgs& a, int grid, cudaStream_t s) {
  switch (K) {
    case MR_SPMM: k_mr_spmm<XT_, VT, R, MR_SPMM, SIGMA><<<grid, kThreads, 0, s>>>(a); break;
    case MR_CHECK: k_mr_spmm<XT_, VT, R, MR_CHECK, SIGMA><<<grid, kThreads, 0, s>>>(a); break;
    case MR_RESID: k_mr_spmm<XT_, VT, R, MR_RESID, SIGMA><<<grid, kThreads, 0, s>>>(a); break;
  }
}

template <int R>
static void spmm_r(int K, const MArgs& a, bool vc, bool sigma, int grid, cudaStream_t s) {
#if SAD_MINRES_PART == 1
  if (vc) { spmm_k<double2, R, false>(K, a, grid, s); return; }
#endif
  if (sigma) spmm_k<double, R, true>(K, a, grid, s);
  else spmm_k<double, R, false>(K, a, grid, s);
}

#define SAD_R_SWITCH(CALL)          \
  switch (R) {                      \
    case 1: CALL(1); break;         \
    case 2: CALL(2); break;         \
    case 3: CALL(3); break;         \
    case 4: CALL(4); break;         \
    case 5: CALL(5); break;         \
    case 6: CALL(6); break;         \
    case 7: CALL(7); break;         \
    case 8: CALL(8); break;         \
    default: return 1;              \
  }

#if SAD_MINRES_PART == 0
int minres_launch_vec_d(int K, const MArgs& a, int R, int grid, cudaStream_t s)
#else
int minres_launch_vec_z(int K, const MArgs& a, int R, int grid, cudaStream_t s)
#endif
{
#define SAD_VEC(RR) vec_r<RR>(K, a, grid, s)
  SAD_R_SWITCH(SAD_VEC)
#undef SAD_VEC
  count_launches(1);
  return 0;
}

#if SAD_MINRES_PART == 0
int minres_launch_spmm_d(int K, const MArgs& a, int R, bool vc, bool sigma, int grid, cudaStream_t s)
#else
int minres_launch_spmm_z(int K, const MArgs& a, int R, bool vc, bool sigma, int grid, cudaStream_t s)
#endif
{
#if SAD_MINRES_PART == 0
  if (vc) return 1;   // complex matrix values need a complex128 block
#endif
#define SAD_SPMM(RR) spmm_r<RR>(K, a, vc, sigma, grid, s)
  SAD_R_SWITCH(SAD_SPMM)
#undef SAD_SPMM
  count_launches(1);
  return 0;
}

}  // namespace sad
