// sad_verify.cuh -- tall-skinny products over the low-rank factors for the
// verification diagnostics: the power iteration of
// true_residual_norm (adi.py:682-726) applies R = A Z G Y^* C^T + M Z G Y^* B^T
// + f g^* to a vector, i.e. products X^H V and X c with X = Z (n x K) or Y
// (m x K) stored row-major.  Both kernels stream X once (HBM-bound).
#pragma once

#include "sad_kernels.cuh"

namespace sad {

// conj(x) * v + acc for a real or complex factor entry and a complex vector entry
__device__ __forceinline__ double2 hfma(double x, double2 v, double2 acc) {
  return make_double2(fma(x, v.x, acc.x), fma(x, v.y, acc.y));
}
__device__ __forceinline__ double2 hfma(double2 x, double2 v, double2 acc) { return cfma(x, v, acc); }
// x * c + acc
__device__ __forceinline__ double2 xfma(double x, double2 c, double2 acc) {
  return make_double2(fma(x, c.x, acc.x), fma(x, c.y, acc.y));
}
__device__ __forceinline__ double2 xfma(double2 x, double2 c, double2 acc) { return fma_(x, c, acc); }

// part[blockIdx][col * S + s] = sum_{rows of this block} conj(X[i, col]) V[i, s].
// Thread (rg, cw): rows rg, rg + RG, ... of the slab, columns cw, cw + CW, ...
// Partial sums over rg are combined through shared memory in a fixed order.
template <typename XT, int S>
__global__ void __launch_bounds__(256) k_ts_hgemv(long long n, long long K, long long ldx,
                                                  const XT* __restrict__ X,
                                                  const double2* __restrict__ V,
                                                  long long rows_per_block, int CW,
                                                  double2* __restrict__ part) {
  __shared__ double2 s_acc[256 * S];
  const int RG = blockDim.x / CW;
  const int cw = threadIdx.x % CW, rg = threadIdx.x / CW;
  const long long r0 = (long long)blockIdx.x * rows_per_block;
  const long long r1 = min(n, r0 + rows_per_block);
  for (long long c0 = 0; c0 < K; c0 += CW) {
    const long long col = c0 + cw;
    double2 acc[S];
#pragma unroll
    for (int s = 0; s < S; ++s) acc[s] = make_double2(0.0, 0.0);
    if (rg < RG && col < K) {
      long long i = r0 + rg;
      for (; i + 3 * RG < r1; i += 4 * RG) {
        XT x[4];
        double2 v[4][S];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          x[q] = X[(i + q * RG) * ldx + col];
#pragma unroll
          for (int s = 0; s < S; ++s) v[q][s] = __ldg(V + (i + q * RG) * S + s);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int s = 0; s < S; ++s) acc[s] = hfma(x[q], v[q][s], acc[s]);
      }
      for (; i < r1; i += RG) {
        const XT x = X[i * ldx + col];
#pragma unroll
        for (int s = 0; s < S; ++s) acc[s] = hfma(x, __ldg(V + i * S + s), acc[s]);
      }
    }
#pragma unroll
    for (int s = 0; s < S; ++s) s_acc[threadIdx.x * S + s] = acc[s];
    __syncthreads();
    if (rg == 0 && col < K) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        double2 t = s_acc[cw * S + s];
        for (int g = 1; g < RG; ++g) t = add(t, s_acc[(g * CW + cw) * S + s]);
        part[(size_t)blockIdx.x * K * S + col * S + s] = t;
      }
    }
    __syncthreads();
  }
}

// out[o] = sum_b part[b][o] in block order (one warp per output, fixed tree).
__global__ void __launch_bounds__(256) k_ts_reduce(const double2* __restrict__ part, int nblocks,
                                                   long long nout, double2* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long o = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (o >= nout) return;
  double2 acc = make_double2(0.0, 0.0);
  for (int b = lane; b < nblocks; b += 32) acc = add(acc, part[(size_t)b * nout + o]);
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) acc = add(acc, shfl_down(acc, sh));
  if (lane == 0) out[o] = acc;
}

// Y[i, s] (+)= sum_col X[i, col] C[col, s]; one warp per row, C staged in shared
// memory; fixed shuffle tree.
template <typename XT, int S>
__global__ void __launch_bounds__(256) k_ts_gemv(long long n, long long K, long long ldx,
                                                 const XT* __restrict__ X,
                                                 const double2* __restrict__ C, double2* Y,
                                                 int accumulate) {
  extern __shared__ double2 s_c[];   // [K][S]
  for (long long o = threadIdx.x; o < K * S; o += blockDim.x) s_c[o] = C[o];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long wpb = blockDim.x >> 5;
  for (long long i = (long long)blockIdx.x * wpb + (threadIdx.x >> 5); i < n;
       i += (long long)gridDim.x * wpb) {
    double2 acc[S];
#pragma unroll
    for (int s = 0; s < S; ++s) acc[s] = make_double2(0.0, 0.0);
    const XT* xr = X + i * ldx;
    for (long long col = lane; col < K; col += 32) {
      const XT x = xr[col];
#pragma unroll
      for (int s = 0; s < S; ++s) acc[s] = xfma(x, s_c[col * S + s], acc[s]);
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
#pragma unroll
      for (int sh = 16; sh > 0; sh >>= 1) acc[s] = add(acc[s], shfl_down(acc[s], sh));
    }
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < S; ++s) Y[i * S + s] = accumulate ? add(Y[i * S + s], acc[s]) : acc[s];
    }
  }
}

}  // namespace sad
