// sad_ring.cuh -- the two basis sweeps of a delayed-Gram CGS2 Arnoldi step as
// stand-alone kernels that stream the basis through a TMA ring (row-partitioned
// engine, large slabs).  They are the persistent kernel's phase-A sweep and
// phase C (sad_persistent.cuh) cut out at its two grid barriers:
//   k_dot_dual_ring   h_raw = V^H w, g_raw = V^H v_j, ||w||^2   (rank-local sums)
//   k_update_ring     w -= V (S c),  ||w||^2
// A block walks row tiles (grid-stride); one stage of the ring = the tile's rows
// of one basis block (cp.async.bulk on an mbarrier, kRingStages deep), the
// per-warp sums of a group of basis blocks go to one of two shared-memory
// buffers by group parity so one block-wide synchronisation per group is enough.
// The direct-load kernels they replace (k_dot_dual, k_update<UPD_ORTH2>) sustain
// ~4 TB/s on config 4; the ring 6-7 TB/s (profiles/r02).
// Outputs (partials layout, last-block reduction into st.rsum) are those of the
// kernels they replace, so the finishers and all-reduces are unchanged.
#pragma once

#include "sad_kernels.cuh"
#include "sad_spmm_bulk.cuh"

namespace sad {

constexpr int kRingStages = 4;
constexpr int kRingGroup = 2;

template <typename XT> __host__ __device__ constexpr int ring_ua() { return sizeof(XT) == 8 ? 8 : 4; }
template <typename XT, int R> __host__ __device__ constexpr int ring_tile_rows() {
  return kWarps * (32 / R) * ring_ua<XT>();
}
template <typename XT, int R> __host__ __device__ constexpr size_t ring_stage_bytes() {
  return ((size_t)ring_tile_rows<XT, R>() * R * sizeof(XT) + 32 + 127) & ~size_t(127);
}
// dynamic shared memory of the two kernels (J <= m + 1 basis blocks)
template <typename XT, int R> __host__ __device__ constexpr size_t ring_dot_smem(int m1) {
  return kRingStages * ring_stage_bytes<XT, R>() + (size_t)2 * m1 * R * sizeof(XT) +
         (size_t)4 * kRingGroup * kWarps * R * sizeof(XT) + (size_t)kWarps * R * 8;
}
template <typename XT, int R> __host__ __device__ constexpr size_t ring_upd_smem(int m1) {
  return kRingStages * ring_stage_bytes<XT, R>() + (size_t)m1 * R * sizeof(XT);
}

template <typename XT, int R>
__global__ void __launch_bounds__(kThreads, 2) k_dot_dual_ring(OrthArgs a) {
  constexpr int GPW = 32 / R, UA = ring_ua<XT>(), T = ring_tile_rows<XT, R>();
  constexpr size_t SB = ring_stage_bytes<XT, R>();
  extern __shared__ __align__(128) unsigned char smem_r[];
  __shared__ __align__(8) unsigned long long s_full[kRingStages];
  __shared__ int s_soff[kRingStages];
  if (*a.st.any_active == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const int j = *a.st.j;
  const int J = j + 1;
  const int m = a.st.m;
  const XT* V = reinterpret_cast<const XT*>(a.V);
  const XT* w = V + (long long)J * a.stride;
  const XT* vj = V + (long long)j * a.stride;
  XT* s_blk = reinterpret_cast<XT*>(smem_r + kRingStages * SB);              // [2J][R]
  XT* s_pw = s_blk + (size_t)2 * (m + 1) * R;                                 // [2][2][group][warps][R]
  double* s_w2 = reinterpret_cast<double*>(s_pw + (size_t)4 * kRingGroup * kWarps * R);
  if (threadIdx.x == 0) {
    for (int q = 0; q < kRingStages; ++q) mbar_init(s_full + q, 1);
    fence_mbar_init();
  }
  for (int o = threadIdx.x; o < 2 * J * R; o += kThreads) s_blk[o] = zero<XT>();
  __syncthreads();
  const long long ntiles = (a.n + T - 1) / T;
  unsigned long long ring = 0;
  unsigned gcount = 0;
  double w2 = 0.0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long base = tile * T;
    const long long nrows = min((long long)T, a.n - base);
    auto issue = [&](int i, int q) {
      const unsigned long long src =
          reinterpret_cast<unsigned long long>(V + (long long)i * a.stride + base * R);
      const unsigned long long e = src + (unsigned long long)(nrows * R) * sizeof(XT);
      const unsigned long long a0 = src & ~15ull, a1 = (e + 15ull) & ~15ull;
      s_soff[q] = (int)((src - a0) / sizeof(XT));
      mbar_expect_tx(s_full + q, (unsigned)(a1 - a0));
      bulk_g2s(smem_r + (size_t)q * SB, reinterpret_cast<const void*>(a0), (unsigned)(a1 - a0),
               s_full + q);
    };
    if (threadIdx.x == 0) {
      fence_proxy_async();
      for (int i = 0; i < min(kRingStages, J); ++i) issue(i, (int)((ring + i) % kRingStages));
    }
    XT wv[UA], xv[UA];
    int lr[UA];
    bool ok[UA];
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      lr[u] = (u * kWarps + warp) * GPW + grp;
      ok[u] = lane_ok && lr[u] < nrows;
      const long long idx = (base + lr[u]) * R + c;
      wv[u] = ok[u] ? w[idx] : zero<XT>();
      xv[u] = ok[u] ? vj[idx] : zero<XT>();
      if (!ok[u]) lr[u] = 0;
      w2 += abs2(wv[u]);
    }
    for (int i0 = 0; i0 < J; i0 += kRingGroup) {
      const int ng = min(kRingGroup, J - i0);
      XT* pw = s_pw + (size_t)(gcount & 1u) * 2 * kRingGroup * kWarps * R;
#pragma unroll
      for (int gi = 0; gi < kRingGroup; ++gi) {
        if (gi < ng) {
          const unsigned long long kk = ring + i0 + gi;
          const int q = (int)(kk % kRingStages);
          mbar_wait(s_full + q, (unsigned)((kk / kRingStages) & 1));
          XT ph = zero<XT>(), pg = zero<XT>();
          if (lane_ok) {
            const XT* Vs = reinterpret_cast<const XT*>(smem_r + (size_t)q * SB) + s_soff[q];
#pragma unroll
            for (int u = 0; u < UA; ++u) {
              const XT v = Vs[lr[u] * R + c];
              ph = cfma(v, wv[u], ph);      // wv / xv are zero for rows outside the tile
              pg = cfma(v, xv[u], pg);
            }
          }
          ph = group_reduce<R>(ph, grp);
          pg = group_reduce<R>(pg, grp);
          if (grp == 0 && lane_ok) {
            pw[(gi * kWarps + warp) * R + c] = ph;
            pw[((kRingGroup + gi) * kWarps + warp) * R + c] = pg;
          }
        }
      }
      __syncthreads();
      if (warp == 0 && lane < R) {
        for (int gi = 0; gi < ng; ++gi) {
          const int i = i0 + gi;
          XT th = s_blk[i * R + lane], tg = s_blk[(J + i) * R + lane];
#pragma unroll
          for (int wq = 0; wq < kWarps; ++wq) {
            th = add(th, pw[(gi * kWarps + wq) * R + lane]);
            tg = add(tg, pw[((kRingGroup + gi) * kWarps + wq) * R + lane]);
          }
          s_blk[i * R + lane] = th;
          s_blk[(J + i) * R + lane] = tg;
        }
      }
      if (threadIdx.x == 0) {
        fence_proxy_async();
        for (int gi = 0; gi < ng; ++gi) {
          const int i = i0 + gi;
          if (i + kRingStages < J) issue(i + kRingStages, (int)((ring + i) % kRingStages));
        }
      }
      ++gcount;
    }
    ring += J;
  }
  w2 = group_reduce<R>(w2, grp);
  if (grp == 0 && lane_ok) s_w2[warp * R + c] = w2;
  __syncthreads();
  // partials and the rank-local reduction: the layout of k_dot_dual
  double* part = a.st.part + (size_t)blockIdx.x * a.st.pstride;
  const int og = 2 * (m + 1) * R, ow = 4 * (m + 1) * R;
  for (int o = threadIdx.x; o < J * R; o += kThreads) {
    const double2 h2c = to_c(s_blk[o]), g2c = to_c(s_blk[J * R + o]);
    part[2 * o] = h2c.x;
    part[2 * o + 1] = h2c.y;
    part[og + 2 * o] = g2c.x;
    part[og + 2 * o + 1] = g2c.y;
  }
  if (threadIdx.x < R) {
    double t = 0.0;
    for (int wq = 0; wq < kWarps; ++wq) t += s_w2[wq * R + threadIdx.x];
    part[ow + threadIdx.x] = t;
  }
  if (last_block(a.st.ticket)) {
    for (int o = threadIdx.x; o < 2 * J * R; o += kThreads) {
      double sh = 0.0, sg = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) {
        const double* pb = a.st.part + (size_t)b * a.st.pstride;
        sh += __ldcg(pb + o);
        sg += __ldcg(pb + og + o);
      }
      a.st.rsum[o] = sh;
      a.st.rsum[og + o] = sg;
    }
    if (threadIdx.x < R) {
      double t = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b)
        t += __ldcg(a.st.part + (size_t)b * a.st.pstride + ow + threadIdx.x);
      a.st.rsum[ow + threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) *a.st.ticket = 0u;
  }
}

// w -= V (S c) with ||w||^2: k_update<UPD_ORTH2> through the ring (coefficients
// st.h2 scaled by S, as there)
template <typename XT, int R>
__global__ void __launch_bounds__(kThreads, 2) k_update_ring(OrthArgs a) {
  constexpr int GPW = 32 / R, UA = ring_ua<XT>(), T = ring_tile_rows<XT, R>();
  constexpr size_t SB = ring_stage_bytes<XT, R>();
  extern __shared__ __align__(128) unsigned char smem_r[];
  __shared__ __align__(8) unsigned long long s_full[kRingStages];
  __shared__ int s_soff[kRingStages];
  __shared__ double s_n[kWarps * 8];
  __shared__ double s_tot[8];
  if (*a.st.any_active == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const int J = *a.st.j + 1;
  const XT* V = reinterpret_cast<const XT*>(a.V);
  XT* w = const_cast<XT*>(V) + (long long)J * a.stride;
  XT* s_coef = reinterpret_cast<XT*>(smem_r + kRingStages * SB);   // [J][R]
  if (threadIdx.x == 0) {
    for (int q = 0; q < kRingStages; ++q) mbar_init(s_full + q, 1);
    fence_mbar_init();
  }
  for (int o = threadIdx.x; o < J * R; o += kThreads) {
    double2 cf = a.st.h2[o];
    const double s = a.st.S[o];
    cf = s == 0.0 ? make_double2(0.0, 0.0) : make_double2(s * cf.x, s * cf.y);
    s_coef[o] = from_c<XT>(cf);
  }
  __syncthreads();
  const long long ntiles = (a.n + T - 1) / T;
  unsigned long long ring = 0;
  double n2 = 0.0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long base = tile * T;
    const long long nrows = min((long long)T, a.n - base);
    auto issue = [&](int i, int q) {
      const unsigned long long src =
          reinterpret_cast<unsigned long long>(V + (long long)i * a.stride + base * R);
      const unsigned long long e = src + (unsigned long long)(nrows * R) * sizeof(XT);
      const unsigned long long a0 = src & ~15ull, a1 = (e + 15ull) & ~15ull;
      s_soff[q] = (int)((src - a0) / sizeof(XT));
      mbar_expect_tx(s_full + q, (unsigned)(a1 - a0));
      bulk_g2s(smem_r + (size_t)q * SB, reinterpret_cast<const void*>(a0), (unsigned)(a1 - a0),
               s_full + q);
    };
    if (threadIdx.x == 0) {
      fence_proxy_async();
      for (int i = 0; i < min(kRingStages, J); ++i) issue(i, (int)((ring + i) % kRingStages));
    }
    XT acc[UA];
    long long idx[UA];
    int lr[UA];
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      lr[u] = (u * kWarps + warp) * GPW + grp;
      idx[u] = (lane_ok && lr[u] < nrows) ? (base + lr[u]) * R + c : -1;
      if (idx[u] < 0) lr[u] = 0;
      acc[u] = zero<XT>();
    }
    for (int i0 = 0; i0 < J; i0 += kRingGroup) {
      const int ng = min(kRingGroup, J - i0);
#pragma unroll
      for (int gi = 0; gi < kRingGroup; ++gi) {
        if (gi < ng) {
          const unsigned long long kk = ring + i0 + gi;
          const int q = (int)(kk % kRingStages);
          mbar_wait(s_full + q, (unsigned)((kk / kRingStages) & 1));
          if (lane_ok) {
            const XT* Vs = reinterpret_cast<const XT*>(smem_r + (size_t)q * SB) + s_soff[q];
            const XT cf = s_coef[(i0 + gi) * R + c];
#pragma unroll
            for (int u = 0; u < UA; ++u) acc[u] = fma_(Vs[lr[u] * R + c], cf, acc[u]);
          }
        }
      }
      __syncthreads();   // the group's stages are consumed
      if (threadIdx.x == 0) {
        fence_proxy_async();
        for (int gi = 0; gi < ng; ++gi) {
          const int i = i0 + gi;
          if (i + kRingStages < J) issue(i + kRingStages, (int)((ring + i) % kRingStages));
        }
      }
    }
    ring += J;
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      if (idx[u] < 0) continue;
      const XT v = sub(w[idx[u]], acc[u]);
      w[idx[u]] = v;
      n2 += abs2(v);
    }
  }
  n2 = group_reduce<R>(n2, grp);
  if (grp == 0 && lane_ok) s_n[warp * R + c] = n2;
  __syncthreads();
  if (threadIdx.x < R) {
    double t = 0.0;
    for (int wq = 0; wq < kWarps; ++wq) t += s_n[wq * R + threadIdx.x];
    a.st.part[(size_t)blockIdx.x * a.st.pstride + threadIdx.x] = t;
  }
  if (last_block(a.st.ticket)) {
    for (int cc = 0; cc < R; ++cc) {
      double t = block_sum_partials(a.st.part, a.st.pstride, gridDim.x, cc);
      if (threadIdx.x == 0) s_tot[cc] = t;
    }
    __syncthreads();
    if (a.st.rsum) {
      if (threadIdx.x < R) a.st.rsum[threadIdx.x] = s_tot[threadIdx.x];
    } else {
      fin_givens(a.st, s_tot);
    }
    if (threadIdx.x == 0) *a.st.ticket = 0u;
  }
}

}  // namespace sad
