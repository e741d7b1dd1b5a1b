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

template <int R>
struct BulkTile {
  static constexpr int GPW = 32 / R;
  static constexpr int U = (128 / (kWarps * GPW)) > 0 ? (128 / (kWarps * GPW)) : 1;
  static constexpr int TR = kWarps * GPW * U;   // rows per tile (~128)
  static constexpr int CAP = 10 * TR;           // staged nonzeros per tile
};

// bytes of dynamic smem for a (VT, R) instantiation
__host__ __device__ constexpr size_t align128(size_t b) { return (b + 127) & ~size_t(127); }
template <int R> __host__ __device__ constexpr size_t bulk_ci_bytes() { return align128((size_t)BulkTile<R>::CAP * 4 + 64); }
template <typename VT, int R> __host__ __device__ constexpr size_t bulk_v_bytes() { return align128((size_t)BulkTile<R>::CAP * sizeof(VT) + 64); }
template <int R> __host__ __device__ constexpr size_t bulk_rp_bytes() { return align128((size_t)(BulkTile<R>::TR + 1) * 4 + 64); }
template <typename VT, int R>
__host__ __device__ constexpr size_t bulk_smem_bytes() {
  return 2 * bulk_ci_bytes<R>() + 2 * bulk_v_bytes<VT, R>() + 3 * bulk_rp_bytes<R>() + 128;
}

// Issue the bulk copy of `count` elements of `esz` bytes starting at element
// `first` of `base`; the source range is widened to 16-byte alignment (arrays
// are padded by the allocator).  Returns the element offset of `first` inside
// the staged buffer and adds the bytes to *tx.
__device__ __forceinline__ int bulk_range(void* dst, const void* base, long long first, long long count,
                                          int esz, unsigned long long* bar, unsigned* tx) {
  const char* b = reinterpret_cast<const char*>(base);
  const unsigned long long a0 = reinterpret_cast<unsigned long long>(b + first * esz) & ~15ull;
  const unsigned long long a1 =
      (reinterpret_cast<unsigned long long>(b + (first + count) * esz) + 15ull) & ~15ull;
  const unsigned bytes = (unsigned)(a1 - a0);
  if (bytes) bulk_g2s(dst, reinterpret_cast<const void*>(a0), bytes, bar);
  *tx += bytes;
  return (int)((reinterpret_cast<unsigned long long>(b + first * esz) - a0) / esz);
}

template <typename XT, typename VT, int R, int MODE, bool PRE, bool SIGMA>
__global__ void __launch_bounds__(kThreads) k_spmm_bulk(SpmmArgs<XT> a) {
  using T = BulkTile<R>;
  constexpr int GPW = T::GPW, U = T::U, TR = T::TR, CAP = T::CAP;
  extern __shared__ __align__(128) unsigned char smem_b[];
  // layout: ci[2][CAP+16] | vals[2][CAP+16] | rp[3][TR+1+16] | bars
  int* s_ci[2];
  VT* s_v[2];
  int* s_rp[3];
  unsigned char* p = smem_b;
  for (int q = 0; q < 2; ++q) { s_ci[q] = reinterpret_cast<int*>(p); p += bulk_ci_bytes<R>(); }
  for (int q = 0; q < 2; ++q) { s_v[q] = reinterpret_cast<VT*>(p); p += bulk_v_bytes<VT, R>(); }
  for (int q = 0; q < 3; ++q) { s_rp[q] = reinterpret_cast<int*>(p); p += bulk_rp_bytes<R>(); }
  unsigned long long* bar_cv = reinterpret_cast<unsigned long long*>((reinterpret_cast<size_t>(p) + 15) & ~size_t(15));
  unsigned long long* bar_rp = bar_cv + 2;
  __shared__ int s_rp_off[3];
  __shared__ int s_cv_off[2][2];   // [buf][ci offset, val offset]
  __shared__ int s_kb[2];
  __shared__ int s_staged[2];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const VT* vals = reinterpret_cast<const VT*>(a.vals);
  const long long ntiles = (a.n + TR - 1) / TR;
  const long long G = gridDim.x;
  const long long K = ntiles > blockIdx.x ? (ntiles - blockIdx.x + G - 1) / G : 0;
  const XT* x = a.x;
  XT* y = a.y;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 2; ++q) mbar_init(bar_cv + q, 1);
    for (int q = 0; q < 3; ++q) mbar_init(bar_rp + q, 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto tile_row0 = [&](long long k) { return (blockIdx.x + k * G) * (long long)TR; };
  auto issue_rp = [&](long long k) {
    const long long r0 = tile_row0(k);
    const long long cnt = min((long long)TR, a.n - r0) + 1;
    unsigned tx = 0;
    const int buf = (int)(k % 3);
    // expect_tx must be armed before the bytes can land: compute the byte count first
    const unsigned long long a0 = reinterpret_cast<unsigned long long>(a.rowptr + r0) & ~15ull;
    const unsigned long long a1 = (reinterpret_cast<unsigned long long>(a.rowptr + r0 + cnt) + 15ull) & ~15ull;
    mbar_expect_tx(bar_rp + buf, (unsigned)(a1 - a0));
    s_rp_off[buf] = bulk_range(s_rp[buf], a.rowptr, r0, cnt, 4, bar_rp + buf, &tx);
  };
  auto issue_cv = [&](long long k) {
    const int rb = (int)(k % 3), cb = (int)(k % 2);
    const long long r0 = tile_row0(k);
    const int rows = (int)min((long long)TR, a.n - r0);
    const int* rp = s_rp[rb] + s_rp_off[rb];
    const int kb = rp[0], ke = rp[rows];
    s_kb[cb] = kb;
    const int nz = ke - kb;
    if (nz + 8 <= CAP) {
      const unsigned long long c0 = reinterpret_cast<unsigned long long>(a.colidx + kb) & ~15ull;
      const unsigned long long c1 = (reinterpret_cast<unsigned long long>(a.colidx + ke) + 15ull) & ~15ull;
      const unsigned long long v0 = reinterpret_cast<unsigned long long>(vals + kb) & ~15ull;
      const unsigned long long v1 = (reinterpret_cast<unsigned long long>(vals + ke) + 15ull) & ~15ull;
      mbar_expect_tx(bar_cv + cb, (unsigned)((c1 - c0) + (v1 - v0)));
      unsigned tx = 0;
      s_cv_off[cb][0] = bulk_range(s_ci[cb], a.colidx, kb, nz, 4, bar_cv + cb, &tx);
      s_cv_off[cb][1] = bulk_range(s_v[cb], vals, kb, nz, (int)sizeof(VT), bar_cv + cb, &tx);
      s_staged[cb] = 1;
    } else {
      s_staged[cb] = 0;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar_cv + cb)) : "memory");
    }
  };

  if (threadIdx.x == 0 && K > 0) {
    issue_rp(0);
    if (K > 1) issue_rp(1);
    mbar_wait(bar_rp + 0, 0);
    issue_cv(0);
  }
  double nacc = 0.0;
  for (long long k = 0; k < K; ++k) {
    const int rb = (int)(k % 3), cb = (int)(k % 2);
    if (threadIdx.x == 0) {
      if (k + 1 < K) {
        mbar_wait(bar_rp + (int)((k + 1) % 3), (unsigned)(((k + 1) / 3) & 1));
        issue_cv(k + 1);
      }
      if (k + 2 < K) issue_rp(k + 2);
    }
    mbar_wait(bar_rp + rb, (unsigned)((k / 3) & 1));
    mbar_wait(bar_cv + cb, (unsigned)((k / 2) & 1));
    __syncthreads();   // s_staged / offsets written by thread 0 are visible
    const long long r0 = tile_row0(k);
    const int* rp = s_rp[rb] + s_rp_off[rb];
    const bool staged = s_staged[cb] != 0;
    const int kb = s_kb[cb];
    const int* ci = staged ? s_ci[cb] + s_cv_off[cb][0] - kb : a.colidx;
    const VT* vv = staged ? s_v[cb] + s_cv_off[cb][1] - kb : vals;
    if (lane_ok) {
      int k0[U], len[U];
      long long idx[U];
      int maxlen = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int lr = (u * kWarps + warp) * GPW + grp;
        const long long row = r0 + lr;
        if (lr < TR && row < a.n) {
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
      XT acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = zero<XT>();
      constexpr int KB = (U <= 2) ? 8 : 4;     // nonzeros per row per batch
      for (int q = 0; q < maxlen; q += KB) {
        // all gathers of the batch are issued before the first FMA consumes one
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
        if (SIGMA) {
          XT xi = x[idx[u]];
          if (PRE) xi = mul(__ldg(a.dinv + idx[u] / R), xi);
          vres = fma_(from_c<XT>(a.sigma), xi, vres);
        }
        if (MODE == SPMM_RESID || MODE == SPMM_RESID_CYCLE) vres = sub(a.b[idx[u]], vres);
        y[idx[u]] = vres;
        if (MODE == SPMM_RESID_CYCLE) nacc += abs2(vres);
      }
    }
    __syncthreads();      // buffers of tile k are free
    if (threadIdx.x == 0) fence_proxy_async();
  }
  (void)nacc;
}

}  // namespace sad
