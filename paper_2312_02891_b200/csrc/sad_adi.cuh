// sad_adi.cuh -- fused ADI-step epilogue (adi.py:518-530) for the device driver.
//
// One launch per outer step replaces 2 axpys + 6 Gram reductions + 6 host syncs:
//   w += gamma * Mz ;  t += conj(gamma) * C^T y
//   G0 = resA^H resA   (-> r_A = block_residual_norm of the A solve)
//   G1 = resB^H resB   (-> r_B)
//   G2 = Mz^H Mz       (-> ||Mz||_2 for u)
//   G3 = Cty^H Cty     (-> ||C^T y||_2 for v)
//   G4 = w^H w, G5 = t^H t  (updated; -> ||w t^*||_2 and next step's ||w||, ||t||)
// Blocks [0, gA) work on the A side (n rows), [gA, gA+gB) on the B side.
// Partials are output-major; the last block reduces them in block order.
#pragma once

#include "sad_persistent.cuh"

namespace sad {

template <typename XT>
struct EpiArgs {
  long long nA, nB;
  int gA, gB;
  double2 gam;
  const XT* mz;
  const XT* resA;
  XT* w;
  const XT* cty;
  const XT* resB;
  XT* t;
  double2* partT;   // [6*R*R][pT]
  int pT;
  unsigned* ticket;
  double2* out;     // [6][R][R]
};

template <typename XT, int R>
__device__ __forceinline__ void gram_rows(const XT* X, long long n, long long r0, long long step,
                                          XT* acc) {
  for (long long row = r0; row < n; row += step) {
    XT xr[R];
#pragma unroll
    for (int q = 0; q < R; ++q) xr[q] = X[row * R + q];
#pragma unroll
    for (int p = 0; p < R; ++p)
#pragma unroll
      for (int q = 0; q < R; ++q) acc[p * R + q] = cfma(xr[p], xr[q], acc[p * R + q]);
  }
}

template <typename XT, int R>
__device__ __forceinline__ void gram_store(XT* acc, double2* partT, int pT, int gid, int blk,
                                           double2 (*s_w)[R * R]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < R * R; ++q) {
    XT v = acc[q];
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v = add(v, shfl_down(v, s));
    if (lane == 0) s_w[warp][q] = to_c(v);
    acc[q] = zero<XT>();
  }
  __syncthreads();
  if (threadIdx.x < R * R) {
    double2 t = make_double2(0.0, 0.0);
    for (int wq = 0; wq < kWarps; ++wq) t = add(t, s_w[wq][threadIdx.x]);
    partT[(size_t)(gid * R * R + threadIdx.x) * pT + blk] = t;
  }
  __syncthreads();
}

template <typename XT, int R>
__global__ void __launch_bounds__(kThreads) k_adi_epilogue(EpiArgs<XT> a) {
  __shared__ double2 s_w[kWarps][R * R];
  XT acc[R * R];
#pragma unroll
  for (int q = 0; q < R * R; ++q) acc[q] = zero<XT>();
  const bool sideA = (int)blockIdx.x < a.gA;
  const int blk = blockIdx.x;
  const int lb = sideA ? blk : blk - a.gA;
  const int nb = sideA ? a.gA : a.gB;
  const long long n = sideA ? a.nA : a.nB;
  const long long r0 = (long long)lb * kThreads + threadIdx.x;
  const long long step = (long long)nb * kThreads;
  const XT gam = from_c<XT>(sideA ? a.gam : cconj(a.gam));
  const XT* mz = sideA ? a.mz : a.cty;
  const XT* res = sideA ? a.resA : a.resB;
  XT* w = sideA ? a.w : a.t;
  // pass 1: w += gamma * Mz and Gram of the updated w
  for (long long row = r0; row < n; row += step) {
    XT xr[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      xr[q] = fma_(gam, mz[row * R + q], w[row * R + q]);
      w[row * R + q] = xr[q];
    }
#pragma unroll
    for (int p = 0; p < R; ++p)
#pragma unroll
      for (int q = 0; q < R; ++q) acc[p * R + q] = cfma(xr[p], xr[q], acc[p * R + q]);
  }
  gram_store<XT, R>(acc, a.partT, a.pT, sideA ? 4 : 5, blk, s_w);
  // pass 2: Gram of Mz (resp. C^T y)
  gram_rows<XT, R>(mz, n, r0, step, acc);
  gram_store<XT, R>(acc, a.partT, a.pT, sideA ? 2 : 3, blk, s_w);
  // pass 3: Gram of the inner residual
  gram_rows<XT, R>(res, n, r0, step, acc);
  gram_store<XT, R>(acc, a.partT, a.pT, sideA ? 0 : 1, blk, s_w);
  // the last block reduces: output (gid, q) over the blocks of its side
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = warp; o < 6 * R * R; o += kWarps) {
    const int gid = o / (R * R);
    const bool A = (gid % 2 == 0);   // even ids: A side
    const int b0 = A ? 0 : a.gA;
    const int b1 = A ? a.gA : a.gA + a.gB;
    const double2* p = a.partT + (size_t)o * a.pT;
    double2 s = make_double2(0.0, 0.0);
    for (int b = b0 + lane; b < b1; b += 32) s = add(s, __ldcg(p + b));
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) s = add(s, shfl_down(s, sh));
    if (lane == 0) a.out[o] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) *a.ticket = 0u;
}

}  // namespace sad
