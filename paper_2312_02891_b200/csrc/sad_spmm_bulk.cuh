// sad_spmm_bulk.cuh -- shifted SpMM with TMA bulk staging of the CSR slices.
//
// A block walks row tiles (grid-stride).  For every tile, one thread issues
// cp.async.bulk copies (the 1-D TMA path) of the tile's row offsets and of its
// contiguous column-index / value range into shared memory, completing on an
// mbarrier; the offsets of tile k+2 and the nonzeros of tile k+1 are in flight
// while tile k computes, so the only memory latency left on the critical path
// is the gather of x.  Lane groups of R lanes own a row (lane c = column c of
// the block), rows are dealt to warps GPW at a time.  Per row the products are
// summed in increasing column order (scipy's csr_matvec order).
#pragma once

#include "sad_kernels.cuh"

namespace sad {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

#ifndef SAD_BULK_ROWS
#define SAD_BULK_ROWS 64       // target rows per tile (tuned: tools/spmm_tune.cu)
#endif
#ifndef SAD_BULK_STAGES
#define SAD_BULK_STAGES 4      // TMA pipeline depth
#endif
#ifndef SAD_BULK_KB
#define SAD_BULK_KB 5          // nonzeros per row gathered per batch
#endif
#ifndef SAD_BULK_MINB
#define SAD_BULK_MINB 4        // __launch_bounds__ min blocks per SM (register cap)
#endif
template <int R>
struct BulkTile {
  static constexpr int GPW = 32 / R;
  static constexpr int U = (SAD_BULK_ROWS / (kWarps * GPW)) > 0 ? (SAD_BULK_ROWS / (kWarps * GPW)) : 1;
  static constexpr int TR = kWarps * GPW * U;   // rows per tile
  static constexpr int CAP = 10 * TR;           // staged nonzeros per tile
  static constexpr int STAGES = SAD_BULK_STAGES;
};

__host__ __device__ constexpr size_t align128(size_t b) { return (b + 127) & ~size_t(127); }
template <int R> __host__ __device__ constexpr size_t bulk_ci_bytes() { return align128((size_t)BulkTile<R>::CAP * 4 + 64); }
template <typename VT, int R> __host__ __device__ constexpr size_t bulk_v_bytes() { return align128((size_t)BulkTile<R>::CAP * sizeof(VT) + 64); }
template <int R> __host__ __device__ constexpr size_t bulk_rp_bytes() { return align128((size_t)(BulkTile<R>::TR + 1) * 4 + 64); }
template <typename VT, int R>
__host__ __device__ constexpr size_t bulk_stage_bytes() {
  return bulk_ci_bytes<R>() + bulk_v_bytes<VT, R>() + bulk_rp_bytes<R>();
}
template <typename VT, int R>
__host__ __device__ constexpr size_t bulk_smem_bytes() {
  return BulkTile<R>::STAGES * bulk_stage_bytes<VT, R>() + 256;
}

// Byte range [a0, a1) covering elements [first, first+count) widened to 16 B.
__device__ __forceinline__ void aligned_range(const void* base, long long first, long long count,
                                              int esz, unsigned long long& a0, unsigned long long& a1) {
  const char* b = reinterpret_cast<const char*>(base);
  a0 = reinterpret_cast<unsigned long long>(b + first * esz) & ~15ull;
  a1 = (reinterpret_cast<unsigned long long>(b + (first + count) * esz) + 15ull) & ~15ull;
}

// Warp-specialised: warps 0..7 consume tiles, warp 8 is the TMA producer.
// full[s]: armed by the producer with the stage's byte count; empty[s]: one
// arrival per consumer warp when it is done with the stage.
// Register cap: complex blocks with two rows per lane (R >= 7) need more than
// the 56 registers of four blocks per SM.
template <typename XT, int R>
__host__ __device__ constexpr int bulk_min_blocks() {
  return (sizeof(XT) == 16 && BulkTile<R>::U >= 2) ? 2 : SAD_BULK_MINB;
}

template <typename XT, typename VT, int R, int MODE, bool PRE, bool SIGMA>
__global__ void __launch_bounds__(kThreads + 32, bulk_min_blocks<XT, R>()) k_spmm_bulk(SpmmArgs<XT> a) {
  using T = BulkTile<R>;
  constexpr int GPW = T::GPW, U = T::U, TR = T::TR, CAP = T::CAP, S = T::STAGES;
  extern __shared__ __align__(128) unsigned char smem_b[];
  constexpr size_t CI = bulk_ci_bytes<R>(), VB = bulk_v_bytes<VT, R>(), RB = bulk_rp_bytes<R>();
  constexpr size_t SB = CI + VB + RB;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_b + S * SB);
  unsigned long long* empty = full + S;
  __shared__ int s_off[S][3];     // element offsets of the staged ranges (ci, v, rp)
  __shared__ int s_kb[S];
  __shared__ int s_staged[S];

  // Arnoldi mode (multi-kernel and row-partitioned engines): w = S_j Op(D^-1 v_j)
  // from basis block j into block j + 1 (+ the FGMRES Z_j), nothing once every
  // column of the cycle has stopped
  if (MODE == SPMM_ARNOLDI && *a.st.any_active == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const VT* vals = reinterpret_cast<const VT*>(a.vals);
  const long long ntiles = (a.n + TR - 1) / TR;
  const long long G = gridDim.x;
  const long long K = ntiles > blockIdx.x ? (ntiles - blockIdx.x + G - 1) / G : 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, kWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kWarps) {
    // ---------------- producer ----------------
    // The whole warp fetches the row ranges (rowptr at the tile boundaries) of
    // 32 tiles at once, one tile per lane, a batch ahead of their use; lane 0
    // then issues each tile's copies with the range taken by shuffle, so the
    // rowptr round trip is paid once per 32 tiles instead of once per tile.
    auto range = [&](long long kk, int& kb, int& ke) {
      if (kk < K) {
        const long long r0 = (blockIdx.x + kk * G) * (long long)TR;
        const int rows = (int)min((long long)TR, a.n - r0);
        kb = __ldg(a.rowptr + r0);
        ke = __ldg(a.rowptr + r0 + rows);
      }
    };
    int kb_cur = 0, ke_cur = 0, kb_nxt = 0, ke_nxt = 0;
    range(lane, kb_cur, ke_cur);
    range(32 + lane, kb_nxt, ke_nxt);
    for (long long k = 0; k < K; ++k) {
      const int l = (int)(k & 31);
      if (l == 0 && k > 0) {
        kb_cur = kb_nxt;
        ke_cur = ke_nxt;
        range(k + 32 + lane, kb_nxt, ke_nxt);
      }
      const int kb = __shfl_sync(0xffffffffu, kb_cur, l);
      const int ke = __shfl_sync(0xffffffffu, ke_cur, l);
      if (lane == 0) {
        const int st = (int)(k % S);
        const long long r0 = (blockIdx.x + k * G) * (long long)TR;
        const int rows = (int)min((long long)TR, a.n - r0);
        if (k >= S) mbar_wait(empty + st, (unsigned)(((k / S) - 1) & 1));
        const int nz = ke - kb;
        unsigned long long p0, p1, c0, c1, v0, v1;
        aligned_range(a.rowptr, r0, rows + 1, 4, p0, p1);
        const bool stage_cv = nz + 8 <= CAP;
        unsigned bytes = (unsigned)(p1 - p0);
        if (stage_cv) {
          aligned_range(a.colidx, kb, nz, 4, c0, c1);
          aligned_range(vals, kb, nz, (int)sizeof(VT), v0, v1);
          bytes += (unsigned)((c1 - c0) + (v1 - v0));
        }
        unsigned char* base = smem_b + st * SB;
        s_kb[st] = kb;
        s_staged[st] = stage_cv ? 1 : 0;
        s_off[st][2] = (int)((reinterpret_cast<unsigned long long>(a.rowptr + r0) - p0) / 4);
        if (stage_cv) {
          s_off[st][0] = (int)((reinterpret_cast<unsigned long long>(a.colidx + kb) - c0) / 4);
          s_off[st][1] = (int)((reinterpret_cast<unsigned long long>(vals + kb) - v0) / sizeof(VT));
        }
        fence_proxy_async();
        mbar_expect_tx(full + st, bytes);
        bulk_g2s(base + CI + VB, reinterpret_cast<const void*>(p0), (unsigned)(p1 - p0), full + st);
        if (stage_cv) {
          if (c1 > c0) bulk_g2s(base, reinterpret_cast<const void*>(c0), (unsigned)(c1 - c0), full + st);
          if (v1 > v0) bulk_g2s(base + CI, reinterpret_cast<const void*>(v0), (unsigned)(v1 - v0), full + st);
        }
      }
      __syncwarp();
    }
    return;
  }

  // ---------------- consumers ----------------
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const XT* x = a.x;
  XT* y = a.y;
  XT* zout = nullptr;
  double scale = 1.0;
  if (MODE == SPMM_ARNOLDI) {
    const int j = *a.st.j;
    x = a.x + (long long)j * a.stride;
    y = const_cast<XT*>(a.x) + (long long)(j + 1) * a.stride;
    if (a.zout) zout = a.zout + (long long)j * a.stride;
    scale = lane_ok ? a.st.S[j * R + c] : 0.0;
  }
  for (long long k = 0; k < K; ++k) {
    const int st = (int)(k % S);
    mbar_wait(full + st, (unsigned)((k / S) & 1));
    const unsigned char* base = smem_b + st * SB;
    const long long r0 = (blockIdx.x + k * G) * (long long)TR;
    const int* rp = reinterpret_cast<const int*>(base + CI + VB) + s_off[st][2];
    const bool staged = s_staged[st] != 0;
    const int kb = s_kb[st];
    const int* ci = staged ? reinterpret_cast<const int*>(base) + s_off[st][0] - kb : a.colidx;
    const VT* vv = staged ? reinterpret_cast<const VT*>(base + CI) + s_off[st][1] - kb : vals;
    if (lane_ok) {
      int k0[U], len[U];
      long long idx[U];
      int maxlen = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int lr = (u * kWarps + warp) * GPW + grp;
        const long long row = r0 + lr;
        if (row < a.n) {
          idx[u] = row * R + c;
          k0[u] = rp[lr];
          len[u] = rp[lr + 1] - k0[u];
        } else {
          idx[u] = -1;
          k0[u] = 0;
          len[u] = 0;
        }
        maxlen = max(maxlen, len[u]);
      }
      XT acc[U], xd[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u] = zero<XT>();
        // the diagonal x entry (shift term / FGMRES Z), loaded with the gathers
        xd[u] = zero<XT>();
        if ((SIGMA || (MODE == SPMM_ARNOLDI && zout)) && idx[u] >= 0) xd[u] = x[idx[u] + a.row0 * R];
      }
      constexpr int KB = SAD_BULK_KB;
      for (int q = 0; q < maxlen; q += KB) {
        XT xg[U][KB];
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int t = 0; t < KB; ++t) {
            xg[u][t] = zero<XT>();
            if (q + t < len[u]) {
              const int col = ci[k0[u] + q + t];
              xg[u][t] = x[(long long)col * R + c];
              if (PRE) xg[u][t] = mul(__ldg(a.dinv + col), xg[u][t]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int t = 0; t < KB; ++t)
            if (q + t < len[u]) acc[u] = fma_(vv[k0[u] + q + t], xg[u][t], acc[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (idx[u] < 0) continue;
        XT vres = acc[u];
        if (SIGMA || (MODE == SPMM_ARNOLDI && zout)) {
          const long long gidx = idx[u] + a.row0 * R;
          XT xi = xd[u];
          if (PRE) xi = mul(__ldg(a.dinv + gidx / R), xi);
          if (SIGMA) vres = fma_(from_c<XT>(a.sigma), xi, vres);
          if (MODE == SPMM_ARNOLDI && zout) zout[idx[u]] = sscal(scale, xi);
        }
        if (MODE == SPMM_ARNOLDI) vres = sscal(scale, vres);
        if (MODE == SPMM_RESID || MODE == SPMM_RESID_CYCLE) vres = sub(a.b[idx[u]], vres);
        y[idx[u]] = vres;
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + st)) : "memory");
  }
}

}  // namespace sad
