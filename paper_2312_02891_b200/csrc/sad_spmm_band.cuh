// sad_spmm_band.cuh -- shifted SpMM with the x block staged in shared memory.
//
// The gathers of x are what bounds a CSR SpMM on r-column blocks: every
// nonzero is a dependent global load, and a warp can only keep a handful in
// flight (k_spmm_bulk: 4.6 TB/s on config 4 with 36 warps per SM; the same
// loop inside the persistent GMRES kernel, 16 warps per SM: ~1 TB/s).  The
// matrices of this path (finite differences / elements on grids; any banded
// matrix) reference, from a tile of consecutive rows, a few CONTIGUOUS ranges
// of x rows.  So an inspector (sad_band_host.cuh, once per sparsity pattern)
// records for every tile of kBandRows rows
//   * up to kBandMaxRanges ranges [xs, xs + xl) of x rows that cover every column
//     of the tile, and where each lands in a shared-memory row buffer (ro);
//   * the tile's nonzeros in a slot-major padded layout [W][kBandRows] with the
//     column replaced by the 16-bit LOCAL row index into that buffer.
// The kernel is then pure streaming: a producer warp issues, per tile, one
// cp.async.bulk (1-D TMA) per x range, ONE for the tile's values + indices
// (stored back to back in one segment) and ONE for the tile's Jacobi rows (a
// per-operator copy of D^-1 in the tile's local row order) -- the kernel is
// bound by the number of copies per tile, not by their bytes -- S tiles ahead,
// completing on an mbarrier; consumer warps read everything from shared memory with no
// global load on their critical path, no row-length predicates, and write y.
// Per row the products are summed in the CSR (increasing column) order, padded
// slots add v = 0 times the row's own x entry.
// HBM bytes per row: W * (2 + sizeof(VT)) + the x rows of the tile's own range
// once (the far ranges are L2 hits: their rows are some other tile's own rows)
// + the y row -- fewer than the CSR's algorithmic bytes.
#pragma once

#include "sad_spmm_bulk.cuh"

namespace sad {

// rows per tile: chosen per pattern by the inspector (256, 128 or 64: the largest
// whose stage fits three times in shared memory; larger tiles mean fewer, longer
// TMA copies per row -- config 4: 64 rows 4.6 TB/s, 128 rows 5.96, 256 rows 6.6)
constexpr int kBandMaxRanges = 6;    // x ranges per tile
constexpr int kBandMaxStages = 8;

struct __align__(16) BandMeta {      // 64 bytes per tile
  unsigned eoff;                     // first element of the tile's padded segment
  short W;                           // padded row length of the tile
  short nr;                          // ranges in use
  int self_off;                      // local row of the tile's first row
  int xs[kBandMaxRanges];            // first x row of range q
  unsigned short xl[kBandMaxRanges]; // rows in range q
  unsigned short ro[kBandMaxRanges]; // local row of range q (ro == xs mod 2, one spare row between ranges)
  int xrows;                         // local rows in use (the tile's Jacobi rows)
};
static_assert(sizeof(BandMeta) == 64, "BandMeta is one 64-byte record");

struct BandCfg {
  int S;                  // pipeline stages
  unsigned SB;            // bytes per stage
  unsigned offD, offV;    // Jacobi rows, values + indices segment inside a stage (x rows at 0)
};


// U: rows per lane group in flight (independent accumulator chains; the consumers
// run 8 or 16 warps per SM on dependent shared-memory loads, so the instruction-
// level parallelism is what keeps them ahead of the copies): 4 when a tile holds
// four passes of the block, else 2 (config 4, 256-row tiles: U = 2 0.537 ms, 4 0.509 ms)
// PAIR: a real fp64 block with an even number of columns processed as R pairs
// (XT = double2, 16-byte lanes: half the instructions per byte -- the 8-byte-lane
// kernel is instruction-bound, config 4's Arnoldi SpMM 0.96 ms vs 0.52 ms).  Every
// product is then COMPONENTWISE: real matrix values and a real Jacobi diagonal
// (a.dinv points to doubles) times a pair, a real shift, the two columns' own
// scales S -- the same real operations as the unpaired kernel, bit for bit.
__device__ __forceinline__ double2 pscal(double2 s, double2 v) {
  return make_double2(s.x == 0.0 ? 0.0 : s.x * v.x, s.y == 0.0 ? 0.0 : s.y * v.y);
}

// U encodes the consumer shape: U = 2: 8 consumer warps, two rows per lane group in
// flight, two blocks per SM for small stages; U = 4: SIXTEEN consumer warps with two
// rows each (tiles of 256 rows and other one-block-per-SM stages: the consumers are
// bound by dependent shared-memory loads, and with the Jacobi prologue 8 warps per
// SM fell behind the copies -- config 4's Arnoldi SpMM 0.87 ms vs 0.49 ms plain).
template <int U> __host__ __device__ constexpr int band_consumer_warps() { return U >= 4 ? 16 : 8; }

template <typename XT, typename VT, int R, int MODE, bool PRE, bool SIGMA, int U, bool PAIR = false>
__global__ void __launch_bounds__((band_consumer_warps<U>() + 1) * 32, U >= 4 ? 1 : 2)
k_spmm_band(SpmmArgs<XT> a, BandCfg cfg) {
  constexpr int NCW = band_consumer_warps<U>();   // consumer warps; warp NCW produces
  constexpr int UR = 2;                           // rows per lane group in flight
  static_assert(!PAIR || (sizeof(XT) == 16 && sizeof(VT) == 8), "pairs: double2 lanes, real values");
  constexpr int GPW = 32 / R;
  constexpr unsigned DS = PAIR ? 8u : (unsigned)sizeof(XT);   // bytes per Jacobi row
  const int TR = a.band_tr;
  constexpr unsigned RB = R * sizeof(XT);
  extern __shared__ __align__(128) unsigned char smem_b[];
  __shared__ __align__(8) unsigned long long full[kBandMaxStages], empty[kBandMaxStages];
  __shared__ int s_W[kBandMaxStages], s_self[kBandMaxStages];

  if (MODE == SPMM_ARNOLDI && *a.st.any_active == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int S = cfg.S;
  const long long ntiles = (a.n + TR - 1) / TR;
  const long long G = gridDim.x;
  const long long K = ntiles > blockIdx.x ? (ntiles - blockIdx.x + G - 1) / G : 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, NCW);
    }
    fence_mbar_init();
  }
  const XT* x = a.x;
  XT* y = a.y;
  XT* zout = nullptr;
  int jcur = 0;
  if (MODE == SPMM_ARNOLDI) {
    jcur = *a.st.j;
    x = a.x + (long long)jcur * a.stride;
    y = const_cast<XT*>(a.x) + (long long)(jcur + 1) * a.stride;
    if (a.zout) zout = a.zout + (long long)jcur * a.stride;
  }
  __syncthreads();
  const BandMeta* metas = reinterpret_cast<const BandMeta*>(a.band_meta);

  if (warp == NCW) {
    // ---------------- producer ----------------
    // Tile records are fetched 32 at a time, one per lane, a batch ahead of their
    // use, into shared memory.  Per tile every copy has its own lane: lane q < nr
    // the x range q (and, PRE, its Jacobi rows), lane 30 the indices, lane 31 the
    // values -- the address arithmetic runs in parallel and ONE convergent
    // cp.async.bulk instruction issues all of them; lane 0 only waits for the
    // stage to be free and arms the barrier with the byte total.
    __shared__ __align__(16) BandMeta s_meta[2][32];
    auto fetch = [&](long long kk, int buf) {
      if (kk < K) {
        const int4* src = reinterpret_cast<const int4*>(metas + (blockIdx.x + kk * G));
        int4* dst = reinterpret_cast<int4*>(&s_meta[buf][lane]);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = __ldg(src + i);
      }
    };
    fetch(lane, 0);
    fetch(32 + lane, 1);
    __syncwarp();
    for (long long k = 0; k < K; ++k) {
      const int l = (int)(k & 31);
      const int buf = (int)((k >> 5) & 1);
      if (l == 0 && k > 0) {
        // the other buffer's batch is finished with: refill it two batches ahead
        fetch(k + 32 + lane, buf ^ 1);
        __syncwarp();
      }
      const BandMeta& m = s_meta[buf][l];
      const int st = (int)(k % S);
      const int nr = m.nr;
      const unsigned nent = (unsigned)m.W * TR;
      unsigned long long src = 0;
      unsigned len = 0, dst = 0;
      // x ranges: widened, 16-byte aligned copies: source and destination are congruent
      // mod 16 (ro == xs mod 2, 16-aligned bases), spare rows absorb the slack
      if (lane < nr) {
        const unsigned long long s0 = reinterpret_cast<unsigned long long>(x) + (unsigned long long)m.xs[lane] * RB;
        const unsigned long long s1 = s0 + (unsigned long long)m.xl[lane] * RB;
        src = s0 & ~15ull;
        len = (unsigned)(((s1 + 15ull) & ~15ull) - src);
        dst = 16u + (unsigned)m.ro[lane] * RB - (unsigned)(s0 - src);
      } else if (lane == 30) {
        if (PRE) {
          // the tile's Jacobi rows, already in local row order (16-byte aligned: the
          // per-tile stride is even)
          const long long tile = blockIdx.x + k * G;
          src = reinterpret_cast<unsigned long long>(a.band_dinv) +
                (unsigned long long)tile * (unsigned long long)a.band_xstride * DS;
          len = ((unsigned)m.xrows * DS + 15u) & ~15u;
          dst = cfg.offD + 16u;
        }
      } else if (lane == 31) {
        // values then indices of the tile, one segment
        src = reinterpret_cast<unsigned long long>(a.band_seg) +
              (unsigned long long)m.eoff * (unsigned long long)(sizeof(VT) + 2);
        len = nent * (unsigned)(sizeof(VT) + 2);
        dst = cfg.offV;
      }
      unsigned bytes = len;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
      unsigned char* base = smem_b + (size_t)st * cfg.SB;
      if (lane == 0) {
        if (k >= S) mbar_wait(empty + st, (unsigned)(((k / S) - 1) & 1));
        s_W[st] = m.W;
        s_self[st] = m.self_off;
        mbar_expect_tx(full + st, bytes);
      }
      __syncwarp();
      if (len) bulk_g2s(base + dst, reinterpret_cast<const void*>(src), len, full + st);
    }
    return;
  }

  // ---------------- consumers ----------------
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  double scale = 1.0;
  double2 scale2 = make_double2(1.0, 1.0);
  if (MODE == SPMM_ARNOLDI) {
    if (PAIR) {
      if (lane_ok) scale2 = make_double2(a.st.S[jcur * 2 * R + 2 * c], a.st.S[jcur * 2 * R + 2 * c + 1]);
    } else {
      scale = lane_ok ? a.st.S[jcur * R + c] : 0.0;
    }
  }
  // x_l scaled by the Jacobi row l; the result scaled per column
  auto dmul = [&](const unsigned char* dbase, int l, XT v) -> XT {
    if constexpr (PAIR) return mul(reinterpret_cast<const double*>(dbase)[l], v);
    else return mul(reinterpret_cast<const XT*>(dbase)[l], v);
  };
  auto colscale = [&](XT v) -> XT {
    if constexpr (PAIR) return pscal(scale2, v);
    else return sscal(scale, v);
  };
  for (long long k = 0; k < K; ++k) {
    const int st = (int)(k % S);
    mbar_wait(full + st, (unsigned)((k / S) & 1));
    const unsigned char* base = smem_b + (size_t)st * cfg.SB;
    const XT* xs = reinterpret_cast<const XT*>(base + 16);
    const unsigned char* ds = base + cfg.offD + 16;
    const int W = s_W[st], self = s_self[st];
    const VT* sv = reinterpret_cast<const VT*>(base + cfg.offV);
    const unsigned short* si = reinterpret_cast<const unsigned short*>(sv + (size_t)W * TR);
    const long long r0 = (blockIdx.x + k * G) * (long long)TR;
    if (lane_ok) {
      for (int rb = 0; rb < TR; rb += NCW * GPW * UR) {
        int lr[UR];
        bool ok[UR];
        XT acc[UR];
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          lr[u] = rb + (u * NCW + warp) * GPW + grp;
          ok[u] = lr[u] < TR && r0 + lr[u] < a.n;
          if (!ok[u]) lr[u] = 0;
          acc[u] = zero<XT>();
        }
        if (!ok[0] && !ok[UR - 1]) continue;
#pragma unroll 4
        for (int t = 0; t < W; ++t) {
#pragma unroll
          for (int u = 0; u < UR; ++u) {
            const int e = t * TR + lr[u];
            const int l = si[e];
            XT xv = xs[l * R + c];
            if (PRE) xv = dmul(ds, l, xv);
            acc[u] = fma_(sv[e], xv, acc[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          if (!ok[u]) continue;
          const long long idx = (r0 + lr[u]) * R + c;
          XT vres = acc[u];
          if (SIGMA || (MODE == SPMM_ARNOLDI && zout)) {
            const int ls = self + lr[u];
            XT xi = xs[ls * R + c];
            if (PRE) xi = dmul(ds, ls, xi);
            if (SIGMA) {
              if constexpr (PAIR) vres = fma_(a.sigma.x, xi, vres);
              else vres = fma_(from_c<XT>(a.sigma), xi, vres);
            }
            if (MODE == SPMM_ARNOLDI && zout) zout[idx] = colscale(xi);
          }
          if (MODE == SPMM_ARNOLDI) vres = colscale(vres);
          if (MODE == SPMM_RESID || MODE == SPMM_RESID_CYCLE) vres = sub(a.b[idx], vres);
          y[idx] = vres;
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + st)) : "memory");
  }
}

// The values + indices segment of every tile from the operator's CSR values:
// tile t at byte eoff * (sizeof(VT) + 2): [W * TR values][W * TR 16-bit local rows]
// (values 0 and the row's own local index for padding).  One block per tile.
template <typename VT>
__global__ void k_band_segments(long long ntiles, int TR, const BandMeta* __restrict__ meta,
                                const unsigned short* __restrict__ idx, const int* __restrict__ perm,
                                const VT* __restrict__ vals, unsigned char* __restrict__ seg) {
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const unsigned eoff = meta[t].eoff;
    const int nent = (int)meta[t].W * TR;
    unsigned char* base = seg + (size_t)eoff * (sizeof(VT) + 2);
    VT* v = reinterpret_cast<VT*>(base);
    unsigned short* ix = reinterpret_cast<unsigned short*>(base + (size_t)nent * sizeof(VT));
    for (int e = threadIdx.x; e < nent; e += blockDim.x) {
      const int p = perm[eoff + e];
      v[e] = p >= 0 ? vals[p] : zero<VT>();
      ix[e] = idx[eoff + e];
    }
  }
}

// The Jacobi rows of every tile in its local row order: out[t * xstride + l] =
// dinv[lrow[t * xstride + l]] (0 for unused local rows)
template <typename DT>
__global__ void k_band_dinv(long long count, const int* __restrict__ lrow, const DT* __restrict__ dinv,
                            DT* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const int g = lrow[i];
    out[i] = g >= 0 ? dinv[g] : zero<DT>();
  }
}

}  // namespace sad
