// sad_bicg.cu -- instantiation and dispatch of the BiCGstab kernels
// (sad_bicg.cuh).  Compiled once per -DSAD_BICG_PART=<0|1>: fp64 / complex128
// blocks, so the two halves build in parallel.
#include <cuda_runtime.h>

#include "sad_bicg.cuh"

#ifndef SAD_BICG_PART
#error "compile with -DSAD_BICG_PART=<0|1>"
#endif

namespace sad {

void count_launches(long long k);   // sad_capi.cu

#if SAD_BICG_PART == 0
using XT_ = double;
#else
using XT_ = double2;
#endif

template <int R>
static void vec_r(int K, const BArgs& a, int grid, cudaStream_t s) {
  switch (K) {
    case BI_START: k_bi_vec<XT_, R, BI_START><<<grid, kThreads, 0, s>>>(a); break;
    case BI_PUPD: k_bi_vec<XT_, R, BI_PUPD><<<grid, kThreads, 0, s>>>(a); break;
    case BI_SUPD: k_bi_vec<XT_, R, BI_SUPD><<<grid, kThreads, 0, s>>>(a); break;
    case BI_RUPD: k_bi_vec<XT_, R, BI_RUPD><<<grid, kThreads, 0, s>>>(a); break;
    case BI_XUPD: k_bi_vec<XT_, R, BI_XUPD><<<grid, kThreads, 0, s>>>(a); break;
  }
}

template <typename VT, int R, bool SIGMA>
static void spmm_k(int K, const BArgs& a, int grid, cudaStream_t s) {
  switch (K) {
    case BI_SPMM_P: k_bi_spmm<XT_, VT, R, BI_SPMM_P, SIGMA><<<grid, kThreads, 0, s>>>(a); break;
    case BI_SPMM_S: k_bi_spmm<XT_, VT, R, BI_SPMM_S, SIGMA><<<grid, kThreads, 0, s>>>(a); break;
    case BI_RESID: k_bi_spmm<XT_, VT, R, BI_RESID, SIGMA><<<grid, kThreads, 0, s>>>(a); break;
  }
}

template <int R>
static void spmm_r(int K, const BArgs& a, bool vc, bool sigma, int grid, cudaStream_t s) {
#if SAD_BICG_PART == 1
  if (vc) { spmm_k<double2, R, false>(K, a, grid, s); return; }
#endif
  if (sigma) spmm_k<double, R, true>(K, a, grid, s);
  else spmm_k<double, R, false>(K, a, grid, s);
}

#if SAD_BICG_PART == 0
int bicg_launch_vec_d(int K, const BArgs& a, int R, int grid, cudaStream_t s)
#else
int bicg_launch_vec_z(int K, const BArgs& a, int R, int grid, cudaStream_t s)
#endif
{
  switch (R) {
    case 1: vec_r<1>(K, a, grid, s); break;
    case 2: vec_r<2>(K, a, grid, s); break;
    case 3: vec_r<3>(K, a, grid, s); break;
    case 4: vec_r<4>(K, a, grid, s); break;
    case 5: vec_r<5>(K, a, grid, s); break;
    case 6: vec_r<6>(K, a, grid, s); break;
    case 7: vec_r<7>(K, a, grid, s); break;
    case 8: vec_r<8>(K, a, grid, s); break;
    default: return 1;
  }
  count_launches(1);
  return 0;
}

#if SAD_BICG_PART == 0
int bicg_launch_spmm_d(int K, const BArgs& a, int R, bool vc, bool sigma, int grid, cudaStream_t s)
#else
int bicg_launch_spmm_z(int K, const BArgs& a, int R, bool vc, bool sigma, int grid, cudaStream_t s)
#endif
{
#if SAD_BICG_PART == 0
  if (vc) return 1;   // complex matrix values need a complex128 block
#endif
  switch (R) {
    case 1: spmm_r<1>(K, a, vc, sigma, grid, s); break;
    case 2: spmm_r<2>(K, a, vc, sigma, grid, s); break;
    case 3: spmm_r<3>(K, a, vc, sigma, grid, s); break;
    case 4: spmm_r<4>(K, a, vc, sigma, grid, s); break;
    case 5: spmm_r<5>(K, a, vc, sigma, grid, s); break;
    case 6: spmm_r<6>(K, a, vc, sigma, grid, s); break;
    case 7: spmm_r<7>(K, a, vc, sigma, grid, s); break;
    case 8: spmm_r<8>(K, a, vc, sigma, grid, s); break;
    default: return 1;
  }
  count_launches(1);
  return 0;
}

}  // namespace sad
