// sad_persistent.cuh -- the whole GMRES/FGMRES solve as ONE cooperative kernel.
//
// Every block owns a contiguous slab of rows.  One Arnoldi step is two
// streaming phases separated by grid-wide "reduce barriers":
//
//   phase A  w = Op(D^-1 v_j)  (fused shifted SpMM, own rows)
//            h_raw = V^H w  and the delayed Gram column g_raw = V^H v_j
//            (ONE sweep over the basis), ||w||^2
//   -- barrier; the last block reduces the partials in block order and forms
//      G[:, j], h1 = S h_raw, h2 = h1 - G h1, c = h1 + h2, coef = S c --
//   phase C  w <- w - sum_i V_i coef_i  (ONE sweep), ||w||^2
//   -- barrier; the last block does the Hessenberg column, Givens rotation,
//      stopping test (and, at a cycle end, the triangular solve) --
//
// so the basis is streamed twice per step (CGS2 streams it four times) and the
// host is not involved until the solve is over.  At a cycle end the blocks
// update x (phase X), recompute the TRUE residual b - Op x into V_0 (phase R)
// and the last block decides per column whether to restart.
//
// Reductions are deterministic (fixed block order, fixed trees).  Mutable
// shared data is read after a barrier (acquire by thread 0 + bar.sync), or
// with ld.cg.
#pragma once

#include <type_traits>

#include "sad_kernels.cuh"
#include "sad_spmm_bulk.cuh"
#include "sad_spmm_band.cuh"

namespace sad {

constexpr int kStages = 4;   // phase-A TMA ring depth
constexpr int kGroup = 2;    // basis blocks reduced per __syncthreads (kStages = 2 * kGroup)
#ifndef SAD_KSTAGES_A1
#define SAD_KSTAGES_A1 3
#endif
#ifndef SAD_KB1
#define SAD_KB1 5
#endif
constexpr int kStagesA1 = SAD_KSTAGES_A1; // staged-SpMM (sub-phase A1) CSR ring depth

// Sub-phase A1 (large slabs): CSR tiles of kWarps * (32 / R) rows -- one row per
// lane group -- staged by TMA; up to 12 nonzeros per row are staged, denser
// tiles read their nonzeros from global memory.
__host__ __device__ constexpr int a1_tile_rows(int R) { return kWarps * (32 / R); }
__host__ __device__ constexpr size_t a1_al16(size_t b) { return (b + 15) & ~size_t(15); }
__host__ __device__ constexpr size_t a1_rp_bytes(int R) { return a1_al16((size_t)(a1_tile_rows(R) + 1) * 4 + 64); }
__host__ __device__ constexpr size_t a1_ci_bytes(int R) { return a1_al16((size_t)12 * a1_tile_rows(R) * 4 + 64); }
__host__ __device__ constexpr size_t a1_vv_bytes(int R, size_t vsz) { return a1_al16((size_t)12 * a1_tile_rows(R) * vsz + 64); }
__host__ __device__ constexpr size_t a1_stage_bytes(int R, size_t vsz) {
  return (a1_rp_bytes(R) + a1_ci_bytes(R) + a1_vv_bytes(R, vsz) + 127) & ~size_t(127);
}

struct PState {
  GState g;              // j, any_active, active, done, kdim, iters, S, H, cs, sn, g, ycoef, ...
  double2* G;            // [R][(m+1)*(m+1)] Gram of the raw-scaled basis
  double2* hc;           // [(m+1)*R] Hessenberg column before rotation
  double2* coef;         // [(m+1)*R] phase-C coefficients
  double2* red;          // [(2(m+1)+1)*R] reduced partials
  unsigned* bar_count;
  unsigned* bar_gen;
  int* err;              // barrier timeout flag
  double* stats;         // [16] bytes_alg, steps, cycles, t_A, t_C, t_X, t_R (ns, block 0),
                         // work_A, work_C (block 0 before arrive), fin_A, fin_C (last block)
  double spmm_bytes_arn; // algorithmic bytes of one Arnoldi SpMM
  double spmm_bytes_res; // algorithmic bytes of one residual SpMM
};

template <typename XT>
struct PArgs {
  long long n;
  const int* rowptr;
  const int* colidx;
  const void* vals;
  const XT* dinv;
  double2 sigma;
  const XT* b;
  XT* x;
  XT* V;
  XT* Z;
  long long stride;      // n*R elements per basis block
  long long rows_per_block;
  int direct_rows;        // direct phase A: staged rows per block (shared-memory capacity)
  int pT;                // block stride of the output-major partials
  int prof;              // record phase timers
  int g_smem;            // stage the Gram block in shared memory (fits)
  int stage_bytes;       // bytes of one phase-A TMA stage (128-aligned)
  int direct_a;          // phase A with direct loads and per-warp sums (small slabs)
  int ring_bytes;        // dynamic-smem bytes of the phase-A rings (basis / A1 CSR)
  int csr_off;           // dynamic-smem byte offset of the resident CSR slab
  int csr_budget;        // bytes available there (0 = CSR read from global)
  int sweep_direct;      // large slabs: basis sweep by basis block with direct loads (no TMA ring)
  int dist_red_min;      // finisher A: partials (outputs x blocks) from which the grid reduces them (SAD_DIST_RED_MIN)
  int ring_c;            // large slabs: phase C through the TMA ring (SAD_RING_C: 0 off, 1 only with
                         // the TMA-ring phase-A sweep, 2 = default: always)
  int dbg_delay_ns;      // tests: the last block idles this long after every phase-C release
  // banded plan for sub-phase A1 (sad_spmm_band.cuh; null: the CSR tiles): rows per
  // block are a multiple of band_tr, the stages live in the ring region
  const void* band_meta;
  const unsigned char* band_seg;   // per tile: values, then 16-bit local row indices
  const void* band_dinv;           // per tile: the Jacobi rows in local row order
  int band_xstride;
  int band_tr;
  BandCfg band_cfg;
  PState st;
};

__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned* p) {
  return *reinterpret_cast<const volatile unsigned*>(p);
}
__device__ __forceinline__ double2 ldcg2(const double2* p) { return __ldcg(p); }
__device__ __forceinline__ double ldcg1(const double* p) { return __ldcg(p); }
__device__ __forceinline__ int ldcgi(const int* p) { return __ldcg(p); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Grid barrier with a reduction slot.  Only thread 0 of a block talks to the
// global counters, with release/acquire semantics at gpu scope; bar.sync makes
// the rest of the block's writes cumulative with thread 0's release, and the
// acquire (which invalidates the SM's L1) orders every later load of the block.
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
  asm volatile("red.add.release.gpu.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Grid barrier.  The arrival counter is zeroed by the host before every launch
// and only ever grows: barrier number k (0-based, counted by every block in
// `narr`) is complete when it reads (k + 1) * gridDim.x, so nothing has to be
// reset between barriers and no block has to look up the current generation
// before it arrives (one L2 round trip less per arrival than a counter + flag
// read pair).  Two uses:
//  * bar_arrive / bar_release / bar_wait: the last block to arrive does a serial
//    finisher and then bumps the generation word the others poll (`gen` is the
//    block's own count of those releases on top of the value at kernel start);
//  * bar_sync: nobody has anything to do before the release, so the waiting
//    blocks poll the arrival counter itself -- the last arrival IS the release.
__device__ __forceinline__ bool bar_arrive(const PState& st, unsigned& narr) {
  __shared__ unsigned s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atom_add_acq_rel(st.bar_count, 1u);
    s_last = (t + 1u == (narr + 1u) * gridDim.x) ? 1u : 0u;
  }
  ++narr;
  __syncthreads();
  return s_last != 0;
}

__device__ __forceinline__ void bar_release(const PState& st, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) red_add_release(st.bar_gen, 1u);
  ++gen;
  __syncthreads();
}

// spin with a 20 s safety timeout (a hang would otherwise wedge the GPU)
template <typename Done>
__device__ __forceinline__ void bar_spin(const PState& st, Done done) {
  unsigned long long t0 = 0;
  unsigned spins = 0;
  while (!done()) {
    if (++spins > 32) __nanosleep(32);
    if ((spins & 4095u) == 0) {
      const unsigned long long t = gtimer();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 20000000000ull) {
        atomicExch(st.err, 1);
        __trap();
      }
    }
  }
}

// Non-last blocks wait for the finisher's release.
__device__ __forceinline__ void bar_wait(const PState& st, unsigned& gen) {
  if (threadIdx.x == 0) {
    const unsigned seen = gen;
    bar_spin(st, [&] { return ld_acquire(st.bar_gen) != seen; });
  }
  ++gen;
  __syncthreads();
}

// Barrier without a finisher.
__device__ __forceinline__ void bar_sync(const PState& st, unsigned& narr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = (narr + 1u) * gridDim.x;
    const unsigned t = atom_add_acq_rel(st.bar_count, 1u);
    if (t + 1u != target)
      bar_spin(st, [&] { return (int)(ld_acquire(st.bar_count) - target) >= 0; });
  }
  ++narr;
  __syncthreads();
}

// Deterministic reduction of per-block partials stored OUTPUT-MAJOR:
// partT[o * pT + b] (complex).  One warp per OB outputs: lane l sums blocks
// l, l+32, ... (coalesced; the KB loads per output of a chunk of 32*KB blocks
// are all issued before the first add, so a chunk costs one L2 round trip),
// then a fixed shuffle tree.
static __device__ void reduce_partials_T(const double2* partT, int pT, int nblocks, int nout,
                                         double2* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int OB = 4;   // outputs per warp
  constexpr int KB = 5;   // 32-block groups per load round (160 blocks)
  for (int o0 = warp * OB; o0 < nout; o0 += kWarps * OB) {
    double2 acc[OB];
#pragma unroll
    for (int q = 0; q < OB; ++q) acc[q] = make_double2(0.0, 0.0);
    for (int b0 = 0; b0 < nblocks; b0 += 32 * KB) {
      double2 v[OB][KB];
#pragma unroll
      for (int q = 0; q < OB; ++q) {
        const double2* p = partT + (size_t)min(o0 + q, nout - 1) * pT;
#pragma unroll
        for (int k = 0; k < KB; ++k) {
          const int b = b0 + k * 32 + lane;
          v[q][k] = (o0 + q < nout && b < nblocks) ? __ldcg(p + b) : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int q = 0; q < OB; ++q)
#pragma unroll
        for (int k = 0; k < KB; ++k) acc[q] = add(acc[q], v[q][k]);
    }
#pragma unroll
    for (int q = 0; q < OB; ++q) {
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) acc[q] = add(acc[q], shfl_down(acc[q], s));
      if (lane == 0 && o0 + q < nout) out[o0 + q] = acc[q];
    }
  }
}

// The same reduction spread over the grid (large J * R * blocks: one block can
// only pull ~100 GB/s out of L2, config 3's 249 x 296 partials took it 16 us per
// Arnoldi step): after a barrier that makes every block's partials visible,
// output o is summed by warp (o / nblocks) of block (o % nblocks) -- lane l adds
// blocks l, l+32, ... in order, then a fixed shuffle tree -- and written to
// red[o]; the finisher then reads nout values instead of nout * nblocks.
static __device__ void reduce_partials_dist(const double2* partT, int pT, int nblocks, int nout,
                                            double2* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int KB = 5;    // 160 blocks per load round
  for (int o = blockIdx.x + warp * nblocks; o < nout; o += kWarps * nblocks) {
    const double2* p = partT + (size_t)o * pT;
    double2 acc = make_double2(0.0, 0.0);
    for (int b0 = 0; b0 < nblocks; b0 += 32 * KB) {
      double2 v[KB];
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const int b = b0 + k * 32 + lane;
        v[k] = b < nblocks ? __ldcg(p + b) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int k = 0; k < KB; ++k) acc = add(acc, v[k]);
    }
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) acc = add(acc, shfl_down(acc, sh));
    if (lane == 0) red[o] = acc;
  }
}

// nout <= 8 outputs: every thread loads its blocks' partials for all outputs
// (one round of independent loads), then a fixed shuffle tree per warp and a
// fixed-order sum over warps.
static __device__ void reduce_partials_small(const double2* partT, int pT, int nblocks, int nout,
                                      double2* out) {
  __shared__ double2 s_ws[kWarps][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2 acc[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) acc[o] = make_double2(0.0, 0.0);
  for (int b = threadIdx.x; b < nblocks; b += kThreads) {
#pragma unroll
    for (int o = 0; o < 8; ++o)
      if (o < nout) acc[o] = add(acc[o], __ldcg(partT + (size_t)o * pT + b));
  }
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    if (o < nout) {
#pragma unroll
      for (int sh = 16; sh > 0; sh >>= 1) acc[o] = add(acc[o], shfl_down(acc[o], sh));
      if (lane == 0) s_ws[warp][o] = acc[o];
    }
  }
  __syncthreads();
  if (threadIdx.x < nout) {
    double2 t = make_double2(0.0, 0.0);
    for (int w = 0; w < kWarps; ++w) t = add(t, s_ws[w][threadIdx.x]);
    out[threadIdx.x] = t;
  }
  __syncthreads();
}

// ----------------------------------------------------------------------------
// the persistent solve kernel
// ----------------------------------------------------------------------------
template <typename XT, typename VT, int R, bool PRE, bool SIGMA, bool FLEX>
__global__ void __launch_bounds__(kThreads, 2) k_gmres_persistent(PArgs<XT> a) {
  constexpr int GPW = 32 / R;
  constexpr int UA = sizeof(XT) == 8 ? 8 : 4;   // rows per lane per phase-A tile
  constexpr int UC = 2;                  // rows per lane per phase-C tile
  constexpr int IB = 4;                  // basis blocks per phase-A round
  extern __shared__ double smem_p[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  PState& st = a.st;
  GState& gs = st.g;
  const int m = gs.m;
  const long long n = a.n;
  const long long r0 = (long long)blockIdx.x * a.rows_per_block;
  const long long r1 = min(n, r0 + a.rows_per_block);
  // rows owned by this lane: r0 + warp*GPW + grp + q*kWarps*GPW
  const long long row_step = (long long)kWarps * GPW;
  const long long row_first = r0 + warp * GPW + grp;
  const int pT = a.pT;
  double2* partT = reinterpret_cast<double2*>(gs.part);
  auto put = [&](int o, double2 v) { partT[(size_t)o * pT + blockIdx.x] = v; };
  unsigned gen = ld_relaxed(st.bar_gen);   // before this block's first arrival: no release yet
  unsigned narr = 0;
  const bool timing = (blockIdx.x == 0 && threadIdx.x == 0);   // counters kept by block 0
  const bool prof = a.prof != 0;                                  // phase timers (profiling)
  unsigned long long tphase = 0;
  double acc_bytes = 0.0, acc_steps = 0.0, acc_cycles = 1.0;
  double t_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // A, C, X, R, workA, workC, spmmA (ns, block 0)

  __shared__ double s_w2[kWarps][8];
  __shared__ int s_any;
  __shared__ double s_Sj[8];     // S_{j+1} of the step just finished (block copy)
  // Per-column Givens state the phase-C finisher reads, kept per block: block 0
  // alone writes gs.active / gs.iters / gs.g, and no grid barrier separates
  // those writes from a late block's reads of the same step, so every block
  // works from its own copy (loaded at the cycle start, after a full barrier,
  // and updated by the identical computation in every block).
  __shared__ int s_cact[8];
  __shared__ long long s_cit[8];
  __shared__ double2 s_cg[8];
  const int cbase = 2 * (m + 1) * R;   // phase-C partial slots (after phase A's)
  // phase-A TMA ring
  __shared__ __align__(8) unsigned long long s_full[kStages];
  __shared__ int s_soff[kStages];
  unsigned long long ring = 0;   // basis-tile copies issued so far (block-uniform)
  // sub-phase A1 CSR ring
  __shared__ __align__(8) unsigned long long s_full1[kStagesA1];
  __shared__ int s_off1[kStagesA1][3], s_kb1[kStagesA1], s_st1[kStagesA1];
  unsigned long long ring1 = 0;
  // sub-phase A1 with a banded plan: tile records (two batches of 32), stage barriers
  // (the records live in dynamic shared memory after the stages: static shared
  // memory stays small -- two blocks of config 3 sit just under the 196 KB
  // carve-out, and the next step, 228 KB, leaves 28 KB of L1 instead of 60 KB,
  // which costs the basis sweeps 17 %)
  __shared__ __align__(8) unsigned long long s_fullb[kBandMaxStages], s_emptyb[kBandMaxStages];
  __shared__ int s_bW[kBandMaxStages], s_bself[kBandMaxStages];
  unsigned long long ringb = 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kStages; ++q) mbar_init(s_full + q, 1);
    for (int q = 0; q < kStagesA1; ++q) mbar_init(s_full1 + q, 1);
    for (int q = 0; q < kBandMaxStages; ++q) {
      mbar_init(s_fullb + q, 1);
      mbar_init(s_emptyb + q, kWarps - 1);
    }
    fence_mbar_init();
  }
  // The block's CSR slab stays in shared memory for the whole solve when it
  // fits (the operator is constant): every SpMM then reads rowptr / colidx /
  // values from shared memory and only gathers x from L2.
  const int* rp_s = nullptr;
  const int* ci_s = nullptr;
  const VT* vv_s = nullptr;
  int kb_s = 0;
  bool csr_s = false;
  if (a.csr_budget > 0 && r1 > r0) {
    kb_s = __ldg(a.rowptr + r0);
    const int nz = __ldg(a.rowptr + r1) - kb_s;
    const size_t rp_b = ((size_t)(r1 - r0 + 1) * 4 + 15) & ~size_t(15);
    const size_t ci_b = ((size_t)nz * 4 + 15) & ~size_t(15);
    if (rp_b + ci_b + (size_t)nz * sizeof(VT) <= (size_t)a.csr_budget) {
      unsigned char* base = reinterpret_cast<unsigned char*>(smem_p) + a.csr_off;
      int* rp_w = reinterpret_cast<int*>(base);
      int* ci_w = reinterpret_cast<int*>(base + rp_b);
      VT* vv_w = reinterpret_cast<VT*>(base + rp_b + ci_b);
      const VT* vals_g = reinterpret_cast<const VT*>(a.vals);
      for (long long i = threadIdx.x; i <= r1 - r0; i += kThreads) rp_w[i] = __ldg(a.rowptr + r0 + i);
      for (int i = threadIdx.x; i < nz; i += kThreads) {
        ci_w[i] = __ldg(a.colidx + kb_s + i);
        vv_w[i] = __ldg(vals_g + kb_s + i);
      }
      rp_s = rp_w;
      ci_s = ci_w;
      vv_s = vv_w;
      csr_s = true;
    }
  }
  __syncthreads();
  // SpMM rows of this block from the resident slab, or from global memory
  auto spmm = [&](auto pre_tag, auto u_tag, const XT* xin, const long long* idx, XT* acc, XT* xi) {
    constexpr bool P = decltype(pre_tag)::value;
    constexpr int U = decltype(u_tag)::value;
    constexpr int SL = (32 / (U * (int)(sizeof(XT) / 8))) < 2 ? 2 : 32 / (U * (int)(sizeof(XT) / 8));
    if (csr_s)
      spmm_rows_s<XT, VT, P, SIGMA, R, U, SL>(rp_s, r0, ci_s, vv_s, kb_s, a.dinv, a.sigma, xin,
                                              idx, c, acc, xi);
    else
      spmm_rows<XT, VT, P, SIGMA, R, U>(a.rowptr, a.colidx, reinterpret_cast<const VT*>(a.vals),
                                        a.dinv, a.sigma, xin, idx, c, acc, xi);
  };

  // ---- init: x = 0, V_0 = b, ||b||^2 -> restart decision --------------------
  {
    if (blockIdx.x == 0 && threadIdx.x < R) {
      gs.iters[threadIdx.x] = 0;
      gs.done[threadIdx.x] = 0;
      gs.active[threadIdx.x] = 0;
      gs.kdim[threadIdx.x] = 0;
    }
    double n2 = 0.0;
    if (lane_ok)
      for (long long row = row_first; row < r1; row += row_step) {
        XT bv = a.b[row * R + c];
        a.V[row * R + c] = bv;
        a.x[row * R + c] = zero<XT>();
        n2 += abs2(bv);
      }
    n2 = group_reduce<R>(n2, grp);
    if (grp == 0 && lane_ok) s_w2[warp][c] = n2;
    __syncthreads();
    if (threadIdx.x < R) {
      double t = 0.0;
      for (int w = 0; w < kWarps; ++w) t += s_w2[w][threadIdx.x];
      put(threadIdx.x, make_double2(t, 0.0));
    }
    if (bar_arrive(st, narr)) {
      reduce_partials_small(partT, pT, gridDim.x, R, st.red);
      __syncthreads();
      __shared__ double s_n2[8];
      if (threadIdx.x < R) s_n2[threadIdx.x] = st.red[threadIdx.x].x;
      __syncthreads();
      // fin_cycle without the host flag protocol
      if (threadIdx.x < R) {
        int cc = threadIdx.x;
        double beta = sqrt(s_n2[cc]);
        gs.beta[cc] = beta;
        bool d = beta <= gs.tol || gs.iters[cc] >= gs.maxit;
        gs.done[cc] = d;
        gs.active[cc] = !d;
        gs.kdim[cc] = 0;
        gs.S[cc] = d ? 0.0 : 1.0 / beta;
        gs.g[cc * (m + 1)] = make_double2(beta, 0.0);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int any = 0;
        for (int cc = 0; cc < R; ++cc) any |= gs.active[cc];
        *gs.any_active = any;
        *gs.j = 0;
      }
      bar_release(st, gen);
    } else {
      bar_wait(st, gen);
    }
  }

  // ---- cycles ---------------------------------------------------------------
  while (true) {
    if (threadIdx.x == 0) s_any = ldcgi(gs.any_active);
    if (threadIdx.x < R) {
      // safe: block 0 rewrites these only after the next phase-A barrier,
      // which this block has not reached yet
      const int cc = threadIdx.x;
      s_cact[cc] = ldcgi(gs.active + cc);
      s_cit[cc] = __ldcg(gs.iters + cc);
      s_cg[cc] = ldcg2(gs.g + (size_t)cc * (m + 1) + ldcgi(gs.j));
    }
    __syncthreads();
    if (!s_any) break;
    // ---------------- Arnoldi steps ----------------
    // j and S_j of the first step of a cycle come from global state (written
    // before a full barrier); later steps use the block's own copies
    int jl = -1;
    while (true) {
      const int j = jl >= 0 ? jl : ldcgi(gs.j);
      const int J = j + 1;
      if (timing) tphase = gtimer();
      // ======== phase A: SpMM + h_raw + delayed Gram column ========
      {
        const XT* vj = a.V + (long long)j * a.stride;
        XT* w = a.V + (long long)J * a.stride;
        const double sj = !lane_ok ? 0.0 : (jl >= 0 ? s_Sj[c] : ldcg1(gs.S + j * R + c));
        // The basis is streamed through a ring of TMA stages (one stage = the
        // tile's rows of one basis block); per basis block the block reduces its
        // h / g contributions through shared memory in a fixed order.
        unsigned char* const smem_c = reinterpret_cast<unsigned char*>(smem_p);
        XT* s_blk = reinterpret_cast<XT*>(smem_c + (size_t)a.ring_bytes);  // [2J][R]
        // per-warp sums of the ring sweep, two buffers by group parity (after s_blk's
        // 2(m+1)R slots): the group after next only overwrites a buffer once warp 0
        // has been through the next group's __syncthreads, so ONE block-wide
        // synchronisation per group is enough
        XT* s_pw = s_blk + (size_t)2 * (m + 1) * R;   // [2][2][kGroup][kWarps][R]
        for (int o = threadIdx.x; o < 2 * J * R; o += kThreads) s_blk[o] = zero<XT>();
        double w2 = 0.0;
        __syncthreads();
        constexpr int T = kWarps * GPW * UA;   // rows per block-tile
        if (a.direct_a) {
          // Small slabs (latency-bound, L2-resident basis): the SpMM writes the
          // block's rows of w (and keeps them and v_j's rows in shared memory);
          // then the basis sweep is split over the warps BY BASIS BLOCK: warp
          // k owns blocks k, k + kWarps, ... and walks all of the block's rows
          // with 8 loads in flight per lane, reading w / v_j from shared
          // memory.  One group reduction per basis block and a single writer per
          // sum (no cross-warp accumulation), so the sweep costs about one L2
          // round trip per basis block a warp owns instead of one per
          // (row tile x group of basis blocks).
          XT* s_wr = s_blk + 2 * J * R;                               // [rows][R]  w
          XT* s_xr = s_wr + (size_t)a.direct_rows * R;                // [rows][R]  v_j
          constexpr int UD = UA / 2;                 // rows per lane per SpMM tile
          constexpr int TD = kWarps * GPW * UD;
          const int nrows_blk = (int)(r1 - r0);
          for (long long base = r0; base < r1; base += TD) {
            const long long nrows = min((long long)TD, r1 - base);
            XT wv[UD], xv[UD];
            long long idx[UD];
#pragma unroll
            for (int u = 0; u < UD; ++u) {
              const int lr = (u * kWarps + warp) * GPW + grp;
              idx[u] = (lane_ok && lr < nrows) ? (base + lr) * R + c : -1;
            }
            const unsigned long long tsp = (timing && prof) ? gtimer() : 0ull;
            spmm(std::integral_constant<bool, PRE>{}, std::integral_constant<int, UD>{}, vj, idx,
                 wv, xv);
            if (timing && prof) t_acc[6] += (double)(gtimer() - tsp);
#pragma unroll
            for (int u = 0; u < UD; ++u) {
              if (idx[u] >= 0) {
                wv[u] = sscal(sj, wv[u]);
                w[idx[u]] = wv[u];
                if (FLEX) {
                  XT zi = PRE ? mul(__ldg(a.dinv + idx[u] / R), xv[u]) : xv[u];
                  a.Z[(long long)j * a.stride + idx[u]] = sscal(sj, zi);
                }
                w2 += abs2(wv[u]);
                const long long lrow = idx[u] - r0 * R;   // (row - r0) * R + c
                s_wr[lrow] = wv[u];
                s_xr[lrow] = xv[u];
              }
            }
          }
          __syncthreads();
          // two basis blocks per warp pass (i and i + kWarps): 2 x KL loads in flight
          for (int i = warp; i < J; i += 2 * kWarps) {
            const int i2 = i + kWarps;
            const bool two = i2 < J;
            const XT* Vi = a.V + (long long)i * a.stride + r0 * R;
            const XT* Vk = a.V + (long long)(two ? i2 : i) * a.stride + r0 * R;
            XT ph = zero<XT>(), pg = zero<XT>(), ph2 = zero<XT>(), pg2 = zero<XT>();
            if (lane_ok) {
              constexpr int KL = 8;
              int rr = grp;
              for (; rr + (KL - 1) * GPW < nrows_blk; rr += KL * GPW) {
                XT vb[KL], vk[KL];
#pragma unroll
                for (int k = 0; k < KL; ++k) {
                  vb[k] = Vi[(rr + k * GPW) * R + c];
                  vk[k] = two ? Vk[(rr + k * GPW) * R + c] : zero<XT>();
                }
#pragma unroll
                for (int k = 0; k < KL; ++k) {
                  const int o = (rr + k * GPW) * R + c;
                  const XT wr = s_wr[o], xr = s_xr[o];
                  ph = cfma(vb[k], wr, ph);
                  pg = cfma(vb[k], xr, pg);
                  ph2 = cfma(vk[k], wr, ph2);
                  pg2 = cfma(vk[k], xr, pg2);
                }
              }
              for (; rr < nrows_blk; rr += GPW) {
                const int o = rr * R + c;
                const XT v = Vi[o];
                const XT v2 = two ? Vk[o] : zero<XT>();
                ph = cfma(v, s_wr[o], ph);
                pg = cfma(v, s_xr[o], pg);
                ph2 = cfma(v2, s_wr[o], ph2);
                pg2 = cfma(v2, s_xr[o], pg2);
              }
            }
            ph = group_reduce<R>(ph, grp);
            pg = group_reduce<R>(pg, grp);
            ph2 = group_reduce<R>(ph2, grp);
            pg2 = group_reduce<R>(pg2, grp);
            if (grp == 0 && lane_ok) {
              s_blk[i * R + c] = ph;
              s_blk[(J + i) * R + c] = pg;
              if (two) {
                s_blk[i2 * R + c] = ph2;
                s_blk[(J + i2) * R + c] = pg2;
              }
            }
          }
        } else {
          // ---- sub-phase A1: w = Op(D^-1 v_j) for the whole slab, CSR tiles
          // staged by TMA (kStagesA1 deep), one row per lane group, 5 gathers of
          // x in flight; w (and Z) written once, read back below from L2 ----
          // ---- sub-phase A1 with a banded plan: the tile's x rows (v_j), Jacobi
          // rows, 16-bit local columns and values staged by TMA, warp 0 issuing
          // every copy of a tile from its own lane; all warps consume from shared
          // memory (sad_spmm_band.cuh) ----
          if (a.band_meta) {
            const unsigned long long tsp = (timing && prof) ? gtimer() : 0ull;
            const int TR = a.band_tr, S1 = a.band_cfg.S;
            constexpr unsigned RB = R * sizeof(XT);
            const BandMeta* metas = reinterpret_cast<const BandMeta*>(a.band_meta) + r0 / TR;
            const long long ntile = r1 > r0 ? (r1 - r0 + TR - 1) / TR : 0;
            BandMeta(*s_bmeta)[32] =
                reinterpret_cast<BandMeta(*)[32]>(smem_c + (size_t)S1 * a.band_cfg.SB);
            auto bfetch = [&](long long kk, int buf) {
              if (kk < ntile) {
                const int4* src = reinterpret_cast<const int4*>(metas + kk);
                int4* dst = reinterpret_cast<int4*>(&s_bmeta[buf][lane]);
#pragma unroll
                for (int i = 0; i < 4; ++i) dst[i] = __ldg(src + i);
              }
            };
            auto bissue = [&](long long t) {   // warp 0, converged
              const BandMeta& m = s_bmeta[(int)((t >> 5) & 1)][(int)(t & 31)];
              const int q = (int)((ringb + t) % S1);
              const unsigned nent = (unsigned)m.W * TR;
              unsigned long long src = 0;
              unsigned len = 0, dst = 0;
              if (lane < m.nr) {
                const unsigned long long s0 = reinterpret_cast<unsigned long long>(vj) + (unsigned long long)m.xs[lane] * RB;
                const unsigned long long s1 = s0 + (unsigned long long)m.xl[lane] * RB;
                src = s0 & ~15ull;
                len = (unsigned)(((s1 + 15ull) & ~15ull) - src);
                dst = 16u + (unsigned)m.ro[lane] * RB - (unsigned)(s0 - src);
              } else if (lane == 30) {
                // the tile's Jacobi rows in local row order (one copy per tile)
                const long long tile = r0 / TR + t;
                src = reinterpret_cast<unsigned long long>(a.band_dinv) +
                      (unsigned long long)tile * (unsigned long long)a.band_xstride * sizeof(XT);
                len = ((unsigned)m.xrows * (unsigned)sizeof(XT) + 15u) & ~15u;
                dst = a.band_cfg.offD + 16u;
              } else if (lane == 31) {
                // values then indices of the tile, one segment
                src = reinterpret_cast<unsigned long long>(a.band_seg) +
                      (unsigned long long)m.eoff * (unsigned long long)(sizeof(VT) + 2);
                len = nent * (unsigned)(sizeof(VT) + 2);
                dst = a.band_cfg.offV;
              }
              unsigned bytes = len;
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
              unsigned char* sb = smem_c + (size_t)q * a.band_cfg.SB;
              if (lane == 0) {
                s_bW[q] = m.W;
                s_bself[q] = m.self_off;
                mbar_expect_tx(s_fullb + q, bytes);
              }
              __syncwarp();
              if (len) bulk_g2s(sb + dst, reinterpret_cast<const void*>(src), len, s_fullb + q);
            };
            // warp 0 produces (runs up to S1 tiles ahead, waiting on the stage's
            // "empty" barrier), warps 1..7 consume: no block-wide synchronisation
            // per tile, the copies of the next tiles are always in flight
            if (warp == 0) {
              bfetch(lane, 0);
              bfetch(32 + lane, 1);
              fence_proxy_async();
              __syncwarp();
              for (long long t = 0; t < ntile; ++t) {
                if ((t & 31) == 0 && t > 0) {
                  bfetch(t + 32 + lane, (int)(((t >> 5) & 1) ^ 1));
                  __syncwarp();
                }
                const unsigned long long kk = ringb + t;
                if (lane == 0 && kk >= (unsigned long long)S1)
                  mbar_wait(s_emptyb + (int)(kk % S1), (unsigned)(((kk / S1) - 1) & 1));
                __syncwarp();
                bissue(t);
              }
            } else {
              constexpr int CW = kWarps - 1;   // consumer warps
              const int cw = warp - 1;
              for (long long t = 0; t < ntile; ++t) {
                const unsigned long long kk = ringb + t;
                const int q = (int)(kk % S1);
                mbar_wait(s_fullb + q, (unsigned)((kk / S1) & 1));
                const unsigned char* sb = smem_c + (size_t)q * a.band_cfg.SB;
                const XT* xs = reinterpret_cast<const XT*>(sb + 16);
                const XT* ds = reinterpret_cast<const XT*>(sb + a.band_cfg.offD + 16);
                const int W = s_bW[q], self = s_bself[q];
                const VT* sv = reinterpret_cast<const VT*>(sb + a.band_cfg.offV);
                const unsigned short* si = reinterpret_cast<const unsigned short*>(sv + (size_t)W * TR);
                const long long row0 = r0 + t * TR;
                if (lane_ok) {
                  constexpr int UB = 2;
                  for (int rb = 0; rb < TR; rb += CW * GPW * UB) {
                    int lr[UB];
                    bool ok[UB];
                    XT acc[UB];
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                      lr[u] = rb + (u * CW + cw) * GPW + grp;
                      ok[u] = lr[u] < TR && row0 + lr[u] < r1;
                      if (!ok[u]) lr[u] = 0;
                      acc[u] = zero<XT>();
                    }
                    if (!ok[0] && !ok[UB - 1]) continue;
#pragma unroll 4
                    for (int tt = 0; tt < W; ++tt) {
#pragma unroll
                      for (int u = 0; u < UB; ++u) {
                        const int e = tt * TR + lr[u];
                        const int l = si[e];
                        XT xv = xs[l * R + c];
                        if (PRE) xv = mul(ds[l], xv);
                        acc[u] = fma_(sv[e], xv, acc[u]);
                      }
                    }
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                      if (!ok[u]) continue;
                      const long long id = (row0 + lr[u]) * R + c;
                      const int ls = self + lr[u];
                      const XT xi = xs[ls * R + c];
                      const XT xsc = PRE ? mul(ds[ls], xi) : xi;
                      XT av = acc[u];
                      if (SIGMA) av = fma_(from_c<XT>(a.sigma), xsc, av);
                      const XT wv1 = sscal(sj, av);
                      w[id] = wv1;
                      if (FLEX) a.Z[(long long)j * a.stride + id] = sscal(sj, xsc);
                      w2 += abs2(wv1);
                    }
                  }
                }
                __syncwarp();
                if (lane == 0)
                  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(s_emptyb + q)) : "memory");
              }
            }
            __syncthreads();   // every tile written before the sweep reads w back
            ringb += (unsigned long long)ntile;
            if (timing && prof) t_acc[6] += (double)(gtimer() - tsp);
          } else
          {
            const unsigned long long tsp = (timing && prof) ? gtimer() : 0ull;
            constexpr int T1 = a1_tile_rows(R);
            constexpr int CAP1 = 12 * T1;
            constexpr size_t CI1 = a1_ci_bytes(R), VV1 = a1_vv_bytes(R, sizeof(VT));
            constexpr size_t SB1 = a1_stage_bytes(R, sizeof(VT));
            const VT* vals_g = reinterpret_cast<const VT*>(a.vals);
            const long long ntile = (r1 - r0 + T1 - 1) / T1;
            // kb/ke of the tile to issue: loaded by the issuing thread one tile
            // ahead (pkb/pke) so the issue at the end of a tile does not wait
            // on a global round trip while the rest of the block is at the
            // tile's __syncthreads
            auto issue1 = [&](long long t, int q, int kb, int ke) {
              const long long row0 = r0 + t * T1;
              const int rows = (int)min((long long)T1, r1 - row0);
              const int nz = ke - kb;
              unsigned long long p0, p1, c0 = 0, c1 = 0, v0 = 0, v1 = 0;
              aligned_range(a.rowptr, row0, rows + 1, 4, p0, p1);
              const bool stg = nz + 8 <= CAP1;
              unsigned bytes = (unsigned)(p1 - p0);
              if (stg) {
                aligned_range(a.colidx, kb, nz, 4, c0, c1);
                aligned_range(vals_g, kb, nz, (int)sizeof(VT), v0, v1);
                bytes += (unsigned)((c1 - c0) + (v1 - v0));
              }
              unsigned char* sb = smem_c + (size_t)q * SB1;
              s_kb1[q] = kb;
              s_st1[q] = stg ? 1 : 0;
              s_off1[q][2] = (int)((reinterpret_cast<unsigned long long>(a.rowptr + row0) - p0) / 4);
              if (stg) {
                s_off1[q][0] = (int)((reinterpret_cast<unsigned long long>(a.colidx + kb) - c0) / 4);
                s_off1[q][1] = (int)((reinterpret_cast<unsigned long long>(vals_g + kb) - v0) / sizeof(VT));
              }
              mbar_expect_tx(s_full1 + q, bytes);
              bulk_g2s(sb + CI1 + VV1, reinterpret_cast<const void*>(p0), (unsigned)(p1 - p0), s_full1 + q);
              if (stg) {
                if (c1 > c0) bulk_g2s(sb, reinterpret_cast<const void*>(c0), (unsigned)(c1 - c0), s_full1 + q);
                if (v1 > v0) bulk_g2s(sb + CI1, reinterpret_cast<const void*>(v0), (unsigned)(v1 - v0), s_full1 + q);
              }
            };
            if (threadIdx.x == 0) {
              fence_proxy_async();
              for (long long t = 0; t < min((long long)kStagesA1, ntile); ++t) {
                const long long row0 = r0 + t * T1;
                const int rows = (int)min((long long)T1, r1 - row0);
                issue1(t, (int)((ring1 + t) % kStagesA1), __ldg(a.rowptr + row0),
                       __ldg(a.rowptr + row0 + rows));
              }
            }
            for (long long t = 0; t < ntile; ++t) {
              const unsigned long long kk = ring1 + t;
              const int q = (int)(kk % kStagesA1);
              // (fp64 blocks only: config 4 -2 %; the complex128 variant is at
              // its register cap and its SpMM got 17 % slower with the prefetch)
              constexpr bool PF = sizeof(XT) == 8;
              int pkb = 0, pke = 0;
              if (PF && threadIdx.x == 0 && t + kStagesA1 < ntile) {
                const long long row0n = r0 + (t + kStagesA1) * T1;
                const int rowsn = (int)min((long long)T1, r1 - row0n);
                pkb = __ldg(a.rowptr + row0n);
                pke = __ldg(a.rowptr + row0n + rowsn);
              }
              mbar_wait(s_full1 + q, (unsigned)((kk / kStagesA1) & 1));
              const long long row0 = r0 + t * T1;
              const int lr = warp * GPW + grp;
              if (lane_ok && row0 + lr < r1) {
                const unsigned char* sb = smem_c + (size_t)q * SB1;
                const int* rp = reinterpret_cast<const int*>(sb + CI1 + VV1) + s_off1[q][2];
                const bool stg = s_st1[q] != 0;
                const int kb = s_kb1[q];
                const int* ci = stg ? reinterpret_cast<const int*>(sb) + s_off1[q][0] - kb : a.colidx;
                const VT* vv = stg ? reinterpret_cast<const VT*>(sb + CI1) + s_off1[q][1] - kb : vals_g;
                const long long row = row0 + lr;
                const long long id = row * R + c;
                const int k0 = rp[lr], k1 = rp[lr + 1];
                XT acc = zero<XT>();
                constexpr int KB1 = SAD_KB1;   // gathers in flight per row
                for (int k = k0; k < k1; k += KB1) {
                  XT xg[KB1];
#pragma unroll
                  for (int tt = 0; tt < KB1; ++tt) {
                    xg[tt] = zero<XT>();
                    if (k + tt < k1) {
                      const int col = ci[k + tt];
                      xg[tt] = vj[(long long)col * R + c];
                      if (PRE) xg[tt] = mul(__ldg(a.dinv + col), xg[tt]);
                    }
                  }
#pragma unroll
                  for (int tt = 0; tt < KB1; ++tt)
                    if (k + tt < k1) acc = fma_(vv[k + tt], xg[tt], acc);
                }
                const XT xi = vj[id];
                const XT xs = PRE ? mul(__ldg(a.dinv + row), xi) : xi;
                if (SIGMA) acc = fma_(from_c<XT>(a.sigma), xs, acc);
                const XT wv1 = sscal(sj, acc);
                w[id] = wv1;
                if (FLEX) a.Z[(long long)j * a.stride + id] = sscal(sj, xs);
                w2 += abs2(wv1);
              }
              __syncthreads();   // stage q consumed
              if (threadIdx.x == 0 && t + kStagesA1 < ntile) {
                fence_proxy_async();
                if (!PF) {
                  const long long row0n = r0 + (t + kStagesA1) * T1;
                  const int rowsn = (int)min((long long)T1, r1 - row0n);
                  pkb = __ldg(a.rowptr + row0n);
                  pke = __ldg(a.rowptr + row0n + rowsn);
                }
                issue1(t + kStagesA1, q, pkb, pke);
              }
            }
            ring1 += (unsigned long long)ntile;
            if (timing && prof) t_acc[6] += (double)(gtimer() - tsp);
          }
          if (a.sweep_direct) {
            // Basis sweep split over the warps BY BASIS BLOCK (as the direct
            // path), w and v_j read back from L2 instead of shared memory: warp
            // k owns blocks k, k + kWarps, ... (two per pass) and walks all of
            // the block's rows with KL rows of loads in flight per lane -- no
            // block-wide synchronisation inside the sweep.
            __syncthreads();   // A1's writes of w visible to the whole block
            const int nrows_blk = (int)(r1 - r0);
            const XT* wg = w + r0 * R;
            const XT* xg = vj + r0 * R;
            for (int i = warp; i < J; i += 2 * kWarps) {
              const int i2 = i + kWarps;
              const bool two = i2 < J;
              const XT* Vi = a.V + (long long)i * a.stride + r0 * R;
              const XT* Vk = a.V + (long long)(two ? i2 : i) * a.stride + r0 * R;
              XT ph = zero<XT>(), pg = zero<XT>(), ph2 = zero<XT>(), pg2 = zero<XT>();
              if (lane_ok) {
                constexpr int KL = sizeof(XT) == 8 ? 8 : 4;
                int rr = grp;
                for (; rr + (KL - 1) * GPW < nrows_blk; rr += KL * GPW) {
                  XT vb[KL], vk[KL], wr[KL], xr[KL];
#pragma unroll
                  for (int k = 0; k < KL; ++k) {
                    const int o = (rr + k * GPW) * R + c;
                    vb[k] = Vi[o];
                    vk[k] = two ? Vk[o] : zero<XT>();
                    wr[k] = wg[o];
                    xr[k] = xg[o];
                  }
#pragma unroll
                  for (int k = 0; k < KL; ++k) {
                    ph = cfma(vb[k], wr[k], ph);
                    pg = cfma(vb[k], xr[k], pg);
                    ph2 = cfma(vk[k], wr[k], ph2);
                    pg2 = cfma(vk[k], xr[k], pg2);
                  }
                }
                for (; rr < nrows_blk; rr += GPW) {
                  const int o = rr * R + c;
                  const XT v = Vi[o];
                  const XT v2 = two ? Vk[o] : zero<XT>();
                  const XT wr = wg[o], xr = xg[o];
                  ph = cfma(v, wr, ph);
                  pg = cfma(v, xr, pg);
                  ph2 = cfma(v2, wr, ph2);
                  pg2 = cfma(v2, xr, pg2);
                }
              }
              ph = group_reduce<R>(ph, grp);
              pg = group_reduce<R>(pg, grp);
              ph2 = group_reduce<R>(ph2, grp);
              pg2 = group_reduce<R>(pg2, grp);
              if (grp == 0 && lane_ok) {
                s_blk[i * R + c] = ph;
                s_blk[(J + i) * R + c] = pg;
                if (two) {
                  s_blk[i2 * R + c] = ph2;
                  s_blk[(J + i2) * R + c] = pg2;
                }
              }
            }
          } else {
          unsigned gcount = 0;   // groups so far: the parity of the per-warp sum buffers
          for (long long base = r0; base < r1; base += T) {
            const long long nrows = min((long long)T, r1 - base);
            auto issue = [&](int i, int q) {
              const unsigned long long src =
                  reinterpret_cast<unsigned long long>(a.V + (long long)i * a.stride + base * R);
              const unsigned long long e = src + (unsigned long long)(nrows * R) * sizeof(XT);
              const unsigned long long a0 = src & ~15ull, a1 = (e + 15ull) & ~15ull;
              s_soff[q] = (int)((src - a0) / sizeof(XT));
              mbar_expect_tx(s_full + q, (unsigned)(a1 - a0));
              bulk_g2s(smem_c + (size_t)q * a.stage_bytes, reinterpret_cast<const void*>(a0),
                       (unsigned)(a1 - a0), s_full + q);
            };
            if (threadIdx.x == 0) {
              fence_proxy_async();
              for (int i = 0; i < min(kStages, J); ++i) issue(i, (int)((ring + i) % kStages));
            }
            // the tile's rows of w (from A1) and v_j (overlaps with the first basis copies)
            XT wv[UA], xv[UA];
            long long idx[UA];
            int lr[UA];
  #pragma unroll
            for (int u = 0; u < UA; ++u) {
              lr[u] = (u * kWarps + warp) * GPW + grp;
              const long long row = base + lr[u];
              idx[u] = (lane_ok && lr[u] < nrows) ? row * R + c : -1;
              wv[u] = idx[u] >= 0 ? w[idx[u]] : zero<XT>();
              xv[u] = idx[u] >= 0 ? vj[idx[u]] : zero<XT>();
            }
            // basis blocks in groups of kGroup per __syncthreads (the other half of
            // the ring is in flight meanwhile)
            for (int i0 = 0; i0 < J; i0 += kGroup) {
              const int ng = min(kGroup, J - i0);
              XT ph[kGroup], pg[kGroup];
  #pragma unroll
              for (int gi = 0; gi < kGroup; ++gi) {
                ph[gi] = zero<XT>();
                pg[gi] = zero<XT>();
                if (gi < ng) {
                  const long long kk = ring + i0 + gi;
                  const int q = (int)(kk % kStages);
                  mbar_wait(s_full + q, (unsigned)((kk / kStages) & 1));
                  const XT* Vs =
                      reinterpret_cast<const XT*>(smem_c + (size_t)q * a.stage_bytes) + s_soff[q];
  #pragma unroll
                  for (int u = 0; u < UA; ++u) {
                    if (idx[u] >= 0) {
                      const XT v = Vs[lr[u] * R + c];
                      ph[gi] = cfma(v, wv[u], ph[gi]);
                      pg[gi] = cfma(v, xv[u], pg[gi]);
                    }
                  }
                }
              }
  #pragma unroll
              for (int gi = 0; gi < kGroup; ++gi) {
                if (gi < ng) {
                  const XT h = group_reduce<R>(ph[gi], grp);
                  const XT gq = group_reduce<R>(pg[gi], grp);
                  if (grp == 0 && lane_ok) {
                    XT* pw = s_pw + (size_t)(gcount & 1u) * 2 * kGroup * kWarps * R;
                    pw[(gi * kWarps + warp) * R + c] = h;
                    pw[((kGroup + gi) * kWarps + warp) * R + c] = gq;
                  }
                }
              }
              __syncthreads();
              if (warp == 0 && lane < R) {
                const XT* pw0 = s_pw + (size_t)(gcount & 1u) * 2 * kGroup * kWarps * R;
                for (int gi = 0; gi < ng; ++gi) {
                  const int i = i0 + gi;
                  XT th = s_blk[i * R + lane], tg = s_blk[(J + i) * R + lane];
  #pragma unroll
                  for (int wq = 0; wq < kWarps; ++wq) {
                    th = add(th, pw0[(gi * kWarps + wq) * R + lane]);
                    tg = add(tg, pw0[((kGroup + gi) * kWarps + wq) * R + lane]);
                  }
                  s_blk[i * R + lane] = th;
                  s_blk[(J + i) * R + lane] = tg;
                }
              }
              if (threadIdx.x == 0) {
                fence_proxy_async();
                for (int gi = 0; gi < ng; ++gi) {
                  const int i = i0 + gi;
                  if (i + kStages < J) issue(i + kStages, (int)((ring + i) % kStages));
                }
              }
              ++gcount;
            }
            ring += J;
          }
          }
        }
        w2 = group_reduce<R>(w2, grp);
        if (grp == 0 && lane_ok) s_w2[warp][c] = w2;
        __syncthreads();
        for (int o = threadIdx.x; o < 2 * J * R; o += kThreads) put(o, to_c(s_blk[o]));
        if (threadIdx.x < R) {
          double t = 0.0;
          for (int wq = 0; wq < kWarps; ++wq) t += s_w2[wq][threadIdx.x];
          put(2 * J * R + threadIdx.x, make_double2(t, 0.0));
        }
        if (timing && prof) t_acc[4] += (double)(gtimer() - tphase);
        const int nout = 2 * J * R + R;
        // many partials: reduce them on the whole grid first
        const bool dist_red = (long long)nout * gridDim.x >= a.dist_red_min && gridDim.x > 1;
        if (dist_red) {
          bar_sync(st, narr);
          reduce_partials_dist(partT, pT, gridDim.x, nout, st.red);
        }
        if (bar_arrive(st, narr)) {
          const unsigned long long tfin = (prof && threadIdx.x == 0) ? gtimer() : 0ull;
          // smem: reduced sums | S | h1 | new Gram column | active flags
          double2* s_red = reinterpret_cast<double2*>(smem_p);
          double2* s_h1 = s_red + nout;
          double2* s_gc = s_h1 + J * R;
          double2* s_snr = s_gc + J * R;                            // [R][j] previous rotations
          double* s_S = reinterpret_cast<double*>(s_snr + j * R);
          double* s_csr = s_S + J * R;                              // [R][j]
          int* s_act = reinterpret_cast<int*>(s_csr + j * R);
          double2* s_G = reinterpret_cast<double2*>(
              (reinterpret_cast<uintptr_t>(s_act + 8) + 15) & ~uintptr_t(15));
          const bool gsm = a.g_smem != 0;
          // everything the finisher reads besides the partials, in one round of
          // independent loads issued before the reduction
          for (int o = threadIdx.x; o < J * R; o += kThreads) s_S[o] = ldcg1(gs.S + o);
          if (threadIdx.x < R) s_act[threadIdx.x] = ldcgi(gs.active + threadIdx.x);
          for (int o = threadIdx.x; o < j * R; o += kThreads) {
            const int cc = o / j, ii = o - cc * j;
            s_snr[cc * j + ii] = ldcg2(gs.sn + (size_t)cc * m + ii);
            s_csr[cc * j + ii] = ldcg1(gs.cs + (size_t)cc * m + ii);
          }
          if (gsm) {
            // asynchronous 16-byte copies (L2 -> shared memory, no register in
            // between): a load + store loop waits for every element at its store,
            // one L2 round trip each, 19 per thread on config 3 at j = 40
            for (int o = threadIdx.x; o < R * j * j; o += kThreads) {
              const int cc = o / (j * j), rem = o - cc * j * j, ii = rem / j, l = rem - ii * j;
              cp_async16(s_G + o, st.G + (size_t)cc * (m + 1) * (m + 1) + (size_t)ii * (m + 1) + l);
            }
          }
          if (dist_red) {
            for (int o = threadIdx.x; o < nout; o += kThreads) s_red[o] = ldcg2(st.red + o);
          } else {
            reduce_partials_T(partT, pT, gridDim.x, nout, s_red);
          }
          cp_async_wait_all();
          __syncthreads();
          // new Gram column G[:, j] and h1 = S h_raw
          for (int o = threadIdx.x; o < J * R; o += kThreads) {
            const int ii = o / R, cc = o - ii * R;
            const double si = s_S[o], sjj = s_S[j * R + cc];
            const double2 graw = s_red[J * R + o];
            const double2 gij = (si == 0.0 || sjj == 0.0)
                                    ? make_double2(0.0, 0.0)
                                    : make_double2(si * sjj * graw.x, si * sjj * graw.y);
            s_gc[o] = gij;
            const double2 hr = s_red[o];
            s_h1[o] = si == 0.0 ? make_double2(0.0, 0.0) : make_double2(si * hr.x, si * hr.y);
          }
          __syncthreads();
          // c = 2 h1 - G h1 (old G entries, column/row j from smem); coef = S c.
          // The old G block is staged in smem with one parallel load when it
          // fits (a.g_smem), else read from global.  Four independent partial
          // sums per output, combined in a fixed order.
          for (int o = threadIdx.x; o < J * R; o += kThreads) {
            const int ii = o / R, cc = o - ii * R;
            double2 gh0 = make_double2(0.0, 0.0), gh1 = gh0, gh2 = gh0, gh3 = gh0;
            if (ii < j) {
              const double2* Grow = gsm ? s_G + (size_t)cc * j * j + (size_t)ii * j
                                        : st.G + (size_t)cc * (m + 1) * (m + 1) + (size_t)ii * (m + 1);
              int l = 0;
              for (; l + 3 < j; l += 4) {
                const double2 g0 = Grow[l], g1 = Grow[l + 1], g2 = Grow[l + 2], g3 = Grow[l + 3];
                gh0 = add(gh0, mul(g0, s_h1[l * R + cc]));
                gh1 = add(gh1, mul(g1, s_h1[(l + 1) * R + cc]));
                gh2 = add(gh2, mul(g2, s_h1[(l + 2) * R + cc]));
                gh3 = add(gh3, mul(g3, s_h1[(l + 3) * R + cc]));
              }
              for (; l < j; ++l) gh0 = add(gh0, mul(Grow[l], s_h1[l * R + cc]));
            } else {
              for (int l = 0; l < j; ++l) gh0 = add(gh0, mul(cconj(s_gc[l * R + cc]), s_h1[l * R + cc]));
            }
            double2 gh = add(add(gh0, gh1), add(gh2, gh3));
            gh = add(gh, mul(s_gc[ii * R + cc], s_h1[j * R + cc]));
            const double2 h1 = s_h1[o];
            double2 cv = make_double2(2.0 * h1.x - gh.x, 2.0 * h1.y - gh.y);
            if (!s_act[cc]) cv = make_double2(0.0, 0.0);
            s_red[o] = cv;     // reuse (sums no longer needed): Hessenberg column before rotation
            const double si = s_S[o];
            st.coef[o] = si == 0.0 ? make_double2(0.0, 0.0) : make_double2(si * cv.x, si * cv.y);
          }
          if (prof && threadIdx.x == 0) atomicAdd(st.stats + 10, (double)(gtimer() - tfin));
          // Every block needs only coef for phase C: release now and do this
          // step's bookkeeping off the critical path.  Its global writes (Gram
          // column, ||w_pre||^2, rotated Hessenberg column) are read by later
          // finishers only, which run after this block's next arrive (release).
          bar_release(st, gen);
          for (int o = threadIdx.x; o < J * R; o += kThreads) {
            const int ii = o / R, cc = o - ii * R;
            double2* Gc = st.G + (size_t)cc * (m + 1) * (m + 1);
            Gc[(size_t)ii * (m + 1) + j] = s_gc[o];          // G[i][j]
            Gc[(size_t)j * (m + 1) + ii] = cconj(s_gc[o]);   // G[j][i]
          }
          if (threadIdx.x < R) gs.wpre2[threadIdx.x] = s_red[2 * J * R + threadIdx.x].x;
          // Apply the previous Givens rotations to the new Hessenberg column now
          // (they do not depend on h_{j+1,j}), so the phase-C finisher only has to
          // form the new rotation.
          {
            if (threadIdx.x < R && s_act[threadIdx.x]) {
              const int cc = threadIdx.x;
              double2 x0 = s_red[cc];
              for (int ii = 0; ii < j; ++ii) {
                const double2 x1 = s_red[(ii + 1) * R + cc];
                const double ci = s_csr[cc * j + ii];
                const double2 si = s_snr[cc * j + ii];
                s_red[ii * R + cc] = add(scal(ci, x0), mul(si, x1));
                x0 = sub(scal(ci, x1), mul(cconj(si), x0));
              }
              st.hc[j * R + cc] = x0;   // partially rotated diagonal entry
            }
            __syncthreads();
            for (int o = threadIdx.x; o < j * R; o += kThreads) {
              const int ii = o / R, cc = o - ii * R;
              if (s_act[cc]) gs.H[((size_t)cc * m + j) * (m + 1) + ii] = s_red[o];
            }
            __syncthreads();   // finisher smem is reused by phase C
          }
        } else {
          bar_wait(st, gen);
        }
      }
      if (timing && prof) { unsigned long long t = gtimer(); t_acc[0] += (double)(t - tphase); tphase = t; }
      // ======== phase C: w -= V coef, ||w||^2 -> Givens ========
      {
        XT* w = a.V + (long long)J * a.stride;
        // large slabs with the TMA-ring sweep: the coefficients sit after the ring
        const bool ringC = !a.direct_a && (a.ring_c > 1 || (a.ring_c && !a.sweep_direct));
        XT* s_coef = ringC ? reinterpret_cast<XT*>(reinterpret_cast<unsigned char*>(smem_p) + (size_t)a.ring_bytes)
                           : reinterpret_cast<XT*>(smem_p);
        for (int o = threadIdx.x; o < J * R; o += kThreads) s_coef[o] = from_c<XT>(ldcg2(st.coef + o));
        __syncthreads();
        double n2 = 0.0;
        if (ringC) {
          // The basis is streamed through the phase-A TMA ring (one stage = the
          // tile's rows of one basis block, kStages deep): the update sweep then
          // runs at the rate of the phase-A sweep (config 4: 5.1 -> ~6 TB/s)
          // instead of at what the direct loads of 16 warps per SM sustain.
          unsigned char* const smem_c = reinterpret_cast<unsigned char*>(smem_p);
          constexpr int T = kWarps * GPW * UA;
          for (long long base = r0; base < r1; base += T) {
            const long long nrows = min((long long)T, r1 - base);
            auto issue = [&](int i, int q) {
              const unsigned long long src =
                  reinterpret_cast<unsigned long long>(a.V + (long long)i * a.stride + base * R);
              const unsigned long long e = src + (unsigned long long)(nrows * R) * sizeof(XT);
              const unsigned long long a0 = src & ~15ull, a1 = (e + 15ull) & ~15ull;
              s_soff[q] = (int)((src - a0) / sizeof(XT));
              mbar_expect_tx(s_full + q, (unsigned)(a1 - a0));
              bulk_g2s(smem_c + (size_t)q * a.stage_bytes, reinterpret_cast<const void*>(a0),
                       (unsigned)(a1 - a0), s_full + q);
            };
            if (threadIdx.x == 0) {
              fence_proxy_async();
              for (int i = 0; i < min(kStages, J); ++i) issue(i, (int)((ring + i) % kStages));
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
            for (int i0 = 0; i0 < J; i0 += kGroup) {
              const int ng = min(kGroup, J - i0);
#pragma unroll
              for (int gi = 0; gi < kGroup; ++gi) {
                if (gi < ng) {
                  const unsigned long long kk = ring + i0 + gi;
                  const int q = (int)(kk % kStages);
                  mbar_wait(s_full + q, (unsigned)((kk / kStages) & 1));
                  if (lane_ok) {
                    const XT* Vs =
                        reinterpret_cast<const XT*>(smem_c + (size_t)q * a.stage_bytes) + s_soff[q];
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
                  if (i + kStages < J) issue(i + kStages, (int)((ring + i) % kStages));
                }
              }
            }
            ring += J;
#pragma unroll
            for (int u = 0; u < UA; ++u) {
              if (idx[u] < 0) continue;
              const XT wv = sub(w[idx[u]], acc[u]);
              w[idx[u]] = wv;
              n2 += abs2(wv);
            }
          }
        } else
        for (long long base = r0; base < r1; base += (long long)kWarps * GPW * UC) {
          XT acc[UC];
          long long idx[UC];
#pragma unroll
          for (int u = 0; u < UC; ++u) {
            const long long row = base + ((long long)u * kWarps + warp) * GPW + grp;
            idx[u] = (lane_ok && row < r1) ? row * R + c : -1;
            acc[u] = zero<XT>();
          }
#pragma unroll 8
          for (int i = 0; i < J; ++i) {
            const XT* vi = a.V + (long long)i * a.stride;
            const XT cf = s_coef[i * R + c];
#pragma unroll
            for (int u = 0; u < UC; ++u)
              if (idx[u] >= 0) acc[u] = fma_(vi[idx[u]], cf, acc[u]);
          }
#pragma unroll
          for (int u = 0; u < UC; ++u) {
            if (idx[u] < 0) continue;
            const XT wv = sub(w[idx[u]], acc[u]);
            w[idx[u]] = wv;
            n2 += abs2(wv);
          }
        }
        n2 = group_reduce<R>(n2, grp);
        if (grp == 0 && lane_ok) s_w2[warp][c] = n2;
        __syncthreads();
        if (threadIdx.x < R) {
          double t = 0.0;
          for (int wq = 0; wq < kWarps; ++wq) t += s_w2[wq][threadIdx.x];
          // phase-C sums in their own slots (cbase..): blocks that run ahead
          // into the next phase A overwrite slots 0.. only
          put(cbase + threadIdx.x, make_double2(t, 0.0));
        }
        if (timing && prof) t_acc[5] += (double)(gtimer() - tphase);
        // Every block waits for all partials and then forms the step's Givens
        // rotation itself (same fixed-order reduction everywhere, so every block
        // gets bit-identical values): no serial finisher between the arrival of
        // the last block and the release.  Block 0 alone writes the global
        // state; the other blocks keep what the next step needs (j, S_{j+1},
        // whether the cycle goes on) in shared memory.
        bar_sync(st, narr);
        if (a.dbg_delay_ns > 0 && blockIdx.x == gridDim.x - 1 && gridDim.x > 1) {
          // race stress (tests): block 0 runs ahead and rewrites the global
          // Givens state before this block's finisher runs
          const unsigned long long t0 = gtimer();
          while (gtimer() - t0 < (unsigned long long)a.dbg_delay_ns) {
          }
          __syncthreads();
        }
        {
          const bool w0 = blockIdx.x == 0;
          const unsigned long long tfin = (prof && w0 && threadIdx.x == 0) ? gtimer() : 0ull;
          __shared__ int s_actn[8];
          __shared__ double2 s_nrm[8];
          int act_c = 0;
          long long it_c = 0;
          double wpre_c = 0.0;
          double2 gj_c = make_double2(0.0, 0.0), hjj = gj_c;
          if (threadIdx.x < R) {
            const int cc = threadIdx.x;
            act_c = s_cact[cc];
            it_c = s_cit[cc];
            wpre_c = ldcg1(gs.wpre2 + cc);
            gj_c = s_cg[cc];
            hjj = ldcg2(st.hc + j * R + cc);
          }
          reduce_partials_small(partT + (size_t)cbase * pT, pT, gridDim.x, R, s_nrm);
          if (threadIdx.x < R) {
            const int cc = threadIdx.x;
            s_actn[cc] = 0;
            double snext = 0.0;
            if (act_c) {
              const double hn = sqrt(s_nrm[cc].x);
              double cj; double2 sjv, rj;
              givens(hjj, make_double2(hn, 0.0), cj, sjv, rj);
              const double2 gn = mul(cconj(sjv), gj_c);
              const double2 gnext = make_double2(-gn.x, -gn.y);
              const long long it = it_c + 1;
              const double est = cabs_(gnext);
              snext = hn > 0.0 ? 1.0 / hn : 0.0;
              bool end = (j + 1 == m) || it >= gs.maxit;
              if (!gs.fixed) end = end || est <= gs.tol || hn <= kLucky * sqrt(wpre_c);
              if (w0) {
                gs.cs[(size_t)cc * m + j] = cj;
                gs.sn[(size_t)cc * m + j] = sjv;
                double2* col = gs.H + ((size_t)cc * m + j) * (m + 1);
                col[j] = rj;
                col[j + 1] = make_double2(0.0, 0.0);
                double2* gv = gs.g + (size_t)cc * (m + 1);
                gv[j + 1] = gnext;
                gv[j] = scal(cj, gj_c);
                gs.iters[cc] = it;
                gs.kdim[cc] = j + 1;
                gs.S[(j + 1) * R + cc] = snext;
                if (end) gs.active[cc] = 0;
              }
              s_actn[cc] = end ? 0 : 1;
              s_cact[cc] = end ? 0 : 1;
              s_cit[cc] = it;
              s_cg[cc] = gnext;
            } else if (w0) {
              gs.S[(j + 1) * R + cc] = 0.0;
            }
            s_Sj[cc] = snext;
          }
          __syncthreads();
          int any_now = 0;
          for (int cc = 0; cc < R; ++cc) any_now |= s_actn[cc];
          if (w0 && threadIdx.x == 0) {
            *gs.any_active = any_now;
            *gs.j = j + 1;
          }
          if (any_now == 0) {
            if (w0) {
              __syncthreads();   // block 0's state writes above, visible to its own threads
              // cycle end: back substitution, one warp per column (lanes split the
              // inner products; fixed shuffle tree)
              for (int cc = warp; cc < R; cc += kWarps) {
                const int k = gs.kdim[cc];
                const double2* Hc = gs.H + (size_t)cc * m * (m + 1);
                const double2* gv = gs.g + (size_t)cc * (m + 1);
                double2* yv = reinterpret_cast<double2*>(smem_p) + (size_t)warp * m;
                for (int ii = k - 1; ii >= 0; --ii) {
                  double2 part = make_double2(0.0, 0.0);
                  for (int l = ii + 1 + lane; l < k; l += 32)
                    part = add(part, mul(Hc[(size_t)l * (m + 1) + ii], yv[l]));
#pragma unroll
                  for (int sh = 16; sh > 0; sh >>= 1) part = add(part, shfl_down(part, sh));
                  if (lane == 0) yv[ii] = cdiv(sub(gv[ii], part), Hc[(size_t)ii * (m + 1) + ii]);
                  __syncwarp();
                }
                for (int ii = lane; ii < m; ii += 32) {
                  double2 y = ii < k ? yv[ii] : make_double2(0.0, 0.0);
                  if (!FLEX && ii < k) {
                    const double sc = gs.S[ii * R + cc];
                    y = sc == 0.0 ? make_double2(0.0, 0.0) : make_double2(sc * y.x, sc * y.y);
                  }
                  gs.ycoef[ii * R + cc] = y;
                }
                __syncwarp();
              }
              __syncthreads();
              if (threadIdx.x == 0) {
                int jx = 0;
                for (int cc = 0; cc < R; ++cc) jx = max(jx, gs.kdim[cc]);
                *gs.jx = jx;
              }
            }
            // everyone waits for block 0's back substitution
            bar_sync(st, narr);
          }
          if (prof && w0 && threadIdx.x == 0) atomicAdd(st.stats + 11, (double)(gtimer() - tfin));
          if (threadIdx.x == 0) s_any = any_now;
          jl = j + 1;
        }
      }
      if (timing) {
        if (prof) {
          unsigned long long t = gtimer();
          t_acc[1] += (double)(t - tphase);
          tphase = t;
        }
        acc_steps += 1.0;
        acc_bytes += st.spmm_bytes_arn + (2.0 * J + 2.0) * (double)a.stride * sizeof(XT);
      }
      __syncthreads();
      if (!s_any) break;
    }
    // ---------------- cycle end ----------------
    // phase X: x += D^-1 sum_i V_i ycoef_i   (FGMRES: sum_i Z_i ycoef_i)
    {
      const int jx = ldcgi(gs.jx);
      XT* s_coef = reinterpret_cast<XT*>(smem_p);
      for (int o = threadIdx.x; o < jx * R; o += kThreads) s_coef[o] = from_c<XT>(ldcg2(gs.ycoef + o));
      __syncthreads();
      const XT* B = FLEX ? a.Z : a.V;
      if (lane_ok && jx > 0)
        for (long long row = row_first; row < r1; row += row_step) {
          XT acc = zero<XT>();
          const XT* bp = B + row * R + c;
          for (int i = 0; i < jx; ++i) acc = fma_(bp[(long long)i * a.stride], s_coef[i * R + c], acc);
          XT xv = a.x[row * R + c];
          xv = FLEX ? add(xv, acc) : fma_(__ldg(a.dinv + row), acc, xv);
          a.x[row * R + c] = xv;
        }
      if (timing) acc_bytes += (double)(jx + 2) * (double)a.stride * sizeof(XT) +
                               (FLEX ? 0.0 : (double)n * sizeof(XT));
      bar_sync(st, narr);
    }
    if (timing && prof) { unsigned long long t = gtimer(); t_acc[2] += (double)(t - tphase); tphase = t; }
    // phase R: V_0 = b - Op x, ||.||^2 -> restart decision
    {
      double n2 = 0.0;
      for (long long base = r0; base < r1; base += (long long)kWarps * GPW * UA) {
        long long idx[UA];
        XT acc[UA], xi[UA];
#pragma unroll
        for (int u = 0; u < UA; ++u) {
          const long long row = base + ((long long)u * kWarps + warp) * GPW + grp;
          idx[u] = (lane_ok && row < r1) ? row * R + c : -1;
        }
        spmm(std::integral_constant<bool, false>{}, std::integral_constant<int, UA>{}, a.x, idx,
             acc, xi);
#pragma unroll
        for (int u = 0; u < UA; ++u) {
          if (idx[u] < 0) continue;
          const XT rv = sub(a.b[idx[u]], acc[u]);
          a.V[idx[u]] = rv;
          n2 += abs2(rv);
        }
      }
      n2 = group_reduce<R>(n2, grp);
      if (grp == 0 && lane_ok) s_w2[warp][c] = n2;
      __syncthreads();
      if (threadIdx.x < R) {
        double t = 0.0;
        for (int wq = 0; wq < kWarps; ++wq) t += s_w2[wq][threadIdx.x];
        put(threadIdx.x, make_double2(t, 0.0));
      }
      if (bar_arrive(st, narr)) {
        reduce_partials_small(partT, pT, gridDim.x, R, st.red);
        __syncthreads();
        if (threadIdx.x < R) {
          const int cc = threadIdx.x;
          const double beta = sqrt(st.red[cc].x);
          gs.beta[cc] = beta;
          const bool d = gs.done[cc] || beta <= gs.tol || gs.iters[cc] >= gs.maxit;
          gs.done[cc] = d;
          gs.active[cc] = !d;
          gs.kdim[cc] = 0;
          gs.S[cc] = d ? 0.0 : 1.0 / beta;
          gs.g[cc * (m + 1)] = make_double2(beta, 0.0);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          int any = 0;
          for (int cc = 0; cc < R; ++cc) any |= gs.active[cc];
          *gs.any_active = any;
          *gs.j = 0;
        }
        bar_release(st, gen);
      } else {
        bar_wait(st, gen);
      }
    }
    if (timing) {
      if (prof) {
        unsigned long long t = gtimer();
        t_acc[3] += (double)(t - tphase);
        tphase = t;
      }
      acc_cycles += 1.0;
      acc_bytes += st.spmm_bytes_res;
    }
  }
  if (timing) {
    st.stats[0] += acc_bytes;
    st.stats[1] += acc_steps;
    st.stats[2] += acc_cycles;
    st.stats[3] += t_acc[0];
    st.stats[4] += t_acc[1];
    st.stats[5] += t_acc[2];
    st.stats[6] += t_acc[3];
    st.stats[8] += t_acc[4];
    st.stats[9] += t_acc[5];
    st.stats[12] += t_acc[6];
  }
}

}  // namespace sad
