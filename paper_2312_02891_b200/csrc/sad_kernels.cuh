// sad_kernels.cuh -- sm_100a kernels of the inner-solve hot path.
//
// Everything here is HBM-bandwidth bound fp64 / complex128 work (SpMM on
// r-column blocks, block dots and updates of classical Gram-Schmidt, small
// Hessenberg/Givens bookkeeping); tensor cores do not apply.
//
// Layout: vector blocks are n x R row-major; element (row, c) at row*R + c.
// XT is the element type (double or double2 = interleaved complex128).
// A "group" of R consecutive lanes owns one row (lane c of the group owns
// column c), so a warp reads 32 consecutive elements per load: coalesced.
//
// Cross-block reductions are deterministic: each block writes its partial
// sums in a fixed order, the last block to arrive (atomic ticket) reduces the
// partials in block order and runs the "finisher" (Givens step, restart
// logic), so the inner loop needs no host round trip.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sad {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr double kLucky = 1e-14;   // GMRES lucky breakdown: h_{j+1,j} <= kLucky*||w_pre||

// ----------------------------------------------------------------------------
// scalar helpers (double = real, double2 = complex)
// ----------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ T zero();
template <> __device__ __forceinline__ double zero<double>() { return 0.0; }
template <> __device__ __forceinline__ double2 zero<double2>() { return make_double2(0.0, 0.0); }

__device__ __forceinline__ double add(double a, double b) { return a + b; }
__device__ __forceinline__ double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double sub(double a, double b) { return a - b; }
__device__ __forceinline__ double2 sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// a*b for (real|complex) x (real|complex)
__device__ __forceinline__ double mul(double a, double b) { return a * b; }
__device__ __forceinline__ double2 mul(double a, double2 b) { return make_double2(a * b.x, a * b.y); }
__device__ __forceinline__ double2 mul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc + a*b
__device__ __forceinline__ double fma_(double a, double b, double acc) { return fma(a, b, acc); }
__device__ __forceinline__ double2 fma_(double a, double2 b, double2 acc) {
  return make_double2(fma(a, b.x, acc.x), fma(a, b.y, acc.y));
}
__device__ __forceinline__ double2 fma_(double2 a, double2 b, double2 acc) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
// acc + conj(a)*b
__device__ __forceinline__ double cfma(double a, double b, double acc) { return fma(a, b, acc); }
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  return make_double2(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.x, b.y, fma(-a.y, b.x, acc.y)));
}
__device__ __forceinline__ double abs2(double a) { return a * a; }
__device__ __forceinline__ double abs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double scal(double s, double a) { return s * a; }
__device__ __forceinline__ double2 scal(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
// scale that maps a zero scale to an exact zero (inactive columns stay finite)
template <typename T> __device__ __forceinline__ T sscal(double s, T a) {
  return s == 0.0 ? zero<T>() : scal(s, a);
}
// complex coefficient (double2) to element type
template <typename T> __device__ __forceinline__ T from_c(double2 z);
template <> __device__ __forceinline__ double from_c<double>(double2 z) { return z.x; }
template <> __device__ __forceinline__ double2 from_c<double2>(double2 z) { return z; }
__device__ __forceinline__ double2 to_c(double a) { return make_double2(a, 0.0); }
__device__ __forceinline__ double2 to_c(double2 a) { return a; }

__device__ __forceinline__ double shfl_down(double v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
__device__ __forceinline__ double2 shfl_down(double2 v, int d) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}

// Sum a per-lane value over the groups of a warp (lanes grp*R + c, grp < GPW);
// lanes of group 0 end up with the column sums.  Fixed tree: deterministic.
template <int R, typename T>
__device__ __forceinline__ T group_reduce(T v, int grp) {
  constexpr int GPW = 32 / R;
#pragma unroll
  for (int s = 1; s < GPW; s <<= 1) {
    T o = shfl_down(v, s * R);
    if ((grp & (2 * s - 1)) == 0 && grp + s < GPW) v = add(v, o);
  }
  return v;
}

// complex helpers for the finishers
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cabs_(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  // Smith's algorithm
  if (fabs(b.x) >= fabs(b.y)) {
    double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  } else {
    double r = b.x / b.y, d = b.y + b.x * r;
    return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
  }
}

// Givens rotation, zlartg convention: [c s; -conj(s) c] [f; g] = [r; 0].
__device__ __forceinline__ void givens(double2 f, double2 g, double& c, double2& s, double2& r) {
  double af = cabs_(f), ag = cabs_(g);
  if (ag == 0.0) { c = 1.0; s = make_double2(0.0, 0.0); r = f; return; }
  if (af == 0.0) { c = 0.0; s = make_double2(g.x / ag, -g.y / ag); r = make_double2(ag, 0.0); return; }
  double nrm = hypot(af, ag);
  double2 al = make_double2(f.x / af, f.y / af);
  c = af / nrm;
  s = mul(al, make_double2(g.x / nrm, -g.y / nrm));
  r = make_double2(al.x * nrm, al.y * nrm);
}

// ----------------------------------------------------------------------------
// GMRES device state (pointers into one workspace allocation)
// ----------------------------------------------------------------------------
struct GState {
  int* j;            // index of the newest basis block in the current cycle
  int* any_active;   // any column still iterating in this cycle
  int* jx;           // max Krylov dimension over columns at cycle end
  int* active;       // [R]
  int* done;         // [R]
  int* kdim;         // [R] Krylov dimension of the current cycle
  long long* iters;  // [R]
  double* S;         // [(m+1)*R] scale of raw basis block i, column c (1/norm)
  double2* h;        // [(m+1)*R] CGS pass-1 coefficients
  double2* h2;       // [(m+1)*R] CGS pass-2 coefficients
  double2* H;        // [R][m][m+1] rotated Hessenberg, column-major per column
  double* cs;        // [R][m]
  double2* sn;       // [R][m]
  double2* g;        // [R][m+1]
  double2* ycoef;    // [(m)*R] x-update coefficients
  double* wpre2;     // [R] ||w||^2 before orthogonalisation
  double* beta;      // [R] true residual norms at the last cycle end
  double* part;      // partial sums [maxBlocks][pstride] (complex stored as 2 doubles)
  unsigned* ticket;  // last-block counter
  unsigned long long* stepseq;  // Givens steps executed
  unsigned long long* cycleseq; // cycles finished
  volatile long long* hflag;    // host-mapped: [0]=stepseq [1]=any_active [2]=cycleseq [3]=any_active
  // row-partitioned (multi-rank) solves: the last block of a reducing kernel
  // writes this rank's sums to `rsum` instead of finishing; the sums are
  // all-reduced over the ranks and k_dist_fin finishes on every rank.
  double* rsum;                 // [pstride] rank sums (null: single-rank finishers)
  volatile long long* hist;     // host-mapped [m+1]: (cycleseq << 1 | any_active) per step
  double tol;
  int maxit;
  int m;
  int R;
  int fixed;         // fixed-step mode: never stop a cycle early
  int pstride;       // doubles per block in `part`
};

// last block to arrive returns true (after all partials are visible)
__device__ __forceinline__ bool last_block(unsigned* ticket) {
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}


// Sum partial[b*pstride + off] over b < nb with all threads of the block (fixed
// strided split + fixed tree => deterministic); result returned to every thread.
__device__ __forceinline__ double block_sum_partials(const double* part, int pstride, int nb, int off) {
  __shared__ double s_red[kThreads];
  double t = 0.0;
  for (int b = threadIdx.x; b < nb; b += kThreads) t += __ldcg(part + (size_t)b * pstride + off);
  s_red[threadIdx.x] = t;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) s_red[threadIdx.x] += s_red[threadIdx.x + s];
    __syncthreads();
  }
  double r = s_red[0];
  __syncthreads();
  return r;
}

// ----------------------------------------------------------------------------
// finishers (run by the last block)
// ----------------------------------------------------------------------------
// After the true residual V_0 = b - Op x: restart decision.
static __device__ void fin_cycle(const GState& st, const double* n2) {
  const int R = st.R;
  if (threadIdx.x < R) {
    int c = threadIdx.x;
    double beta = sqrt(n2[c]);
    st.beta[c] = beta;
    bool d = st.done[c] || beta <= st.tol || st.iters[c] >= st.maxit;
    st.done[c] = d ? 1 : 0;
    st.active[c] = d ? 0 : 1;
    st.kdim[c] = 0;
    st.S[c] = d ? 0.0 : 1.0 / beta;
    st.g[c * (st.m + 1)] = make_double2(beta, 0.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int any = 0;
    for (int c = 0; c < R; ++c) any |= st.active[c];
    *st.any_active = any;
    *st.j = 0;
    unsigned long long cs = ++(*st.cycleseq);
    st.hflag[3] = any;
    __threadfence_system();
    st.hflag[2] = (long long)cs;
  }
}

// After pass-2 update with ||w||^2: Hessenberg column, Givens, stopping test.
static __device__ void fin_givens(const GState& st, const double* n2) {
  const int R = st.R, m = st.m;
  const int j = *st.j;
  if (threadIdx.x < R) {
    int c = threadIdx.x;
    if (st.active[c]) {
      double hn = sqrt(n2[c]);
      double2* col = st.H + ((size_t)c * m + j) * (m + 1);
      for (int i = 0; i <= j; ++i) col[i] = add(st.h[i * R + c], st.h2[i * R + c]);
      double* csv = st.cs + (size_t)c * m;
      double2* snv = st.sn + (size_t)c * m;
      for (int i = 0; i < j; ++i) {
        double2 a = col[i], b = col[i + 1];
        double ci = csv[i];
        double2 si = snv[i];
        col[i] = add(scal(ci, a), mul(si, b));
        col[i + 1] = sub(scal(ci, b), mul(cconj(si), a));
      }
      double cj; double2 sj, rj;
      givens(col[j], make_double2(hn, 0.0), cj, sj, rj);
      csv[j] = cj; snv[j] = sj;
      col[j] = rj;
      col[j + 1] = make_double2(0.0, 0.0);
      double2* gv = st.g + (size_t)c * (m + 1);
      double2 gj = gv[j];
      double2 gn = mul(cconj(sj), gj);
      gv[j + 1] = make_double2(-gn.x, -gn.y);
      gv[j] = scal(cj, gj);
      long long it = ++st.iters[c];
      st.kdim[c] = j + 1;
      double est = cabs_(gv[j + 1]);
      st.S[(j + 1) * R + c] = hn > 0.0 ? 1.0 / hn : 0.0;
      bool end = (j + 1 == m) || it >= st.maxit;
      if (!st.fixed) end = end || est <= st.tol || hn <= kLucky * sqrt(st.wpre2[c]);
      if (end) st.active[c] = 0;
    } else {
      st.S[(j + 1) * R + c] = 0.0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int any = 0;
    for (int c = 0; c < R; ++c) any |= st.active[c];
    *st.any_active = any;
    *st.j = j + 1;
    unsigned long long s = ++(*st.stepseq);
    if (st.hist) st.hist[j + 1] = (long long)((*st.cycleseq) << 1) | any;
    st.hflag[1] = any;
    __threadfence_system();
    st.hflag[0] = (long long)s;
  }
}

// U rows at once: the nonzeros are walked in slices of 4 with a warp-lane-local
// trip count, so the (colidx -> x) load chains of different rows and different
// nonzeros are independent and overlap (one row at a time serialises ~2 L2
// round trips per nonzero pair).  Per row the products are still accumulated
// in increasing column order, as scipy's csr_matvec does.
template <typename XT, typename VT, bool PRE, bool SIGMA, int R, int U>
__device__ __forceinline__ void spmm_rows(const int* __restrict__ rowptr,
                                          const int* __restrict__ colidx,
                                          const VT* __restrict__ vals,
                                          const XT* __restrict__ dinv, double2 sigma,
                                          const XT* x, const long long* idx, int c,
                                          XT* acc, XT* xi) {
  int k0[U], len[U];
  int maxlen = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    acc[u] = zero<XT>();
    xi[u] = zero<XT>();
    if (idx[u] >= 0) {
      const long long row = idx[u] / R;
      k0[u] = __ldg(rowptr + row);
      len[u] = __ldg(rowptr + row + 1) - k0[u];
      xi[u] = x[idx[u]];
    } else {
      k0[u] = 0;
      len[u] = 0;
    }
    maxlen = max(maxlen, len[u]);
  }
  for (int q = 0; q < maxlen; q += 4) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (q + t < len[u]) {
          const int kk = k0[u] + q + t;
          const int col = __ldg(colidx + kk);
          const VT v = __ldg(vals + kk);
          XT xv = x[(long long)col * R + c];
          if (PRE) xv = mul(__ldg(dinv + col), xv);
          acc[u] = fma_(v, xv, acc[u]);
        }
      }
    }
  }
  if (SIGMA) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (idx[u] >= 0) {
        const XT xs = PRE ? mul(__ldg(dinv + idx[u] / R), xi[u]) : xi[u];
        acc[u] = fma_(from_c<XT>(sigma), xs, acc[u]);
      }
    }
  }
}

// spmm_rows with the block's CSR slab resident in shared memory (rp_s holds
// rowptr[r0 .. r1], ci_s / vv_s the nonzeros from kb on): only the x gathers
// touch L2, SL of them per row in flight.  Same summation order as spmm_rows.
template <typename XT, typename VT, bool PRE, bool SIGMA, int R, int U, int SL>
__device__ __forceinline__ void spmm_rows_s(const int* rp_s, long long r0, const int* ci_s,
                                            const VT* vv_s, int kb,
                                            const XT* __restrict__ dinv, double2 sigma,
                                            const XT* x, const long long* idx, int c,
                                            XT* acc, XT* xi) {
  int k0[U], len[U];
  int maxlen = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    acc[u] = zero<XT>();
    xi[u] = zero<XT>();
    if (idx[u] >= 0) {
      const int lr = (int)(idx[u] / R - r0);
      k0[u] = rp_s[lr] - kb;
      len[u] = rp_s[lr + 1] - rp_s[lr];
      xi[u] = x[idx[u]];
    } else {
      k0[u] = 0;
      len[u] = 0;
    }
    maxlen = max(maxlen, len[u]);
  }
  for (int q = 0; q < maxlen; q += SL) {
    XT xg[U][SL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int t = 0; t < SL; ++t) {
        xg[u][t] = zero<XT>();
        if (q + t < len[u]) {
          const int col = ci_s[k0[u] + q + t];
          xg[u][t] = x[(long long)col * R + c];
          if (PRE) xg[u][t] = mul(__ldg(dinv + col), xg[u][t]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int t = 0; t < SL; ++t)
        if (q + t < len[u]) acc[u] = fma_(vv_s[k0[u] + q + t], xg[u][t], acc[u]);
  }
  if (SIGMA) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (idx[u] >= 0) {
        const XT xs = PRE ? mul(__ldg(dinv + idx[u] / R), xi[u]) : xi[u];
        acc[u] = fma_(from_c<XT>(sigma), xs, acc[u]);
      }
    }
  }
}

// ----------------------------------------------------------------------------
// Kernel 1: fused shifted SpMM
//   y = scale_c * [ A * (D^-1 x) + sigma * D^-1 x_row ]   (ARNOLDI, PRE)
//   y = A x + sigma x                                      (APPLY)
//   y = b - (A x + sigma x)  [+ ||y_c||^2 -> fin_cycle]    (RESID / RESID_CYCLE)
// A is CSR with VT values (double, or double2 for an assembled complex
// A + sigma M); SIGMA adds the identity-mass shift in the epilogue.
// ----------------------------------------------------------------------------
enum SpmmMode { SPMM_APPLY = 0, SPMM_RESID = 1, SPMM_RESID_CYCLE = 2, SPMM_ARNOLDI = 3 };

template <typename XT>
struct SpmmArgs {
  long long n;
  const int* rowptr;
  const int* colidx;
  const void* vals;
  const XT* x;       // APPLY/RESID input; ARNOLDI: basis base pointer
  XT* y;             // output (ARNOLDI: unused, computed from basis)
  const XT* b;       // RESID rhs
  const XT* dinv;    // Jacobi inverse diagonal (PRE)
  XT* zout;          // FGMRES Z base pointer (ARNOLDI, may be null)
  double2 sigma;
  long long stride;  // elements per basis block (n*R)
  long long row0;    // bulk APPLY/RESID on a row range: global row of local row 0
                     // (rowptr, y, b are offset by the caller; x, dinv are global)
  // banded plan (sad_spmm_band.cuh; null = the CSR kernels): tile records, 16-bit
  // local row indices and values in the padded slot-major layout
  const void* band_meta;
  const unsigned char* band_seg;      // per tile: values, then 16-bit local row indices
  const void* band_dinv;              // per tile: the Jacobi rows in local row order (PRE)
  int band_xstride;                   // local rows reserved per tile in band_dinv
  int band_xcap, band_wmax, band_tr;   // local x rows / padded row length (max), rows per tile
  GState st;
};

template <typename XT, typename VT, int R, int MODE, bool PRE, bool SIGMA>
__global__ void __launch_bounds__(kThreads) k_spmm(SpmmArgs<XT> a) {
  constexpr int GPW = 32 / R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const XT* x = a.x;
  XT* y = a.y;
  XT* zout = nullptr;
  double scale = 1.0;
  if (MODE == SPMM_ARNOLDI) {
    if (*a.st.any_active == 0) return;
    const int j = *a.st.j;
    x = a.x + (long long)j * a.stride;
    y = const_cast<XT*>(a.x) + (long long)(j + 1) * a.stride;
    if (a.zout) zout = a.zout + (long long)j * a.stride;
    scale = lane_ok ? a.st.S[j * R + c] : 0.0;
  }
  const VT* vals = reinterpret_cast<const VT*>(a.vals);
  const XT sig = from_c<XT>(a.sigma);
  double nacc = 0.0;
  const long long rows_per_iter = (long long)gridDim.x * kWarps * GPW;
  (void)sig;
  constexpr int U = 2;   // rows per lane group per iteration (independent load chains)
  if (lane_ok) {
    for (long long row0 = ((long long)blockIdx.x * kWarps + warp) * GPW + grp; row0 < a.n;
         row0 += rows_per_iter * U) {
      long long idx[U];
      XT acc[U], xi[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long row = row0 + u * rows_per_iter;
        idx[u] = row < a.n ? row * R + c : -1;
      }
      spmm_rows<XT, VT, PRE, SIGMA, R, U>(a.rowptr, a.colidx, vals, a.dinv, a.sigma, x, idx,
                                          c, acc, xi);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (idx[u] < 0) continue;
        XT v = acc[u];
        if (MODE == SPMM_ARNOLDI && zout) {
          const XT xs = PRE ? mul(__ldg(a.dinv + idx[u] / R), xi[u]) : xi[u];
          zout[idx[u]] = sscal(scale, xs);
        }
        if (MODE == SPMM_ARNOLDI) v = sscal(scale, v);
        if (MODE == SPMM_RESID || MODE == SPMM_RESID_CYCLE) v = sub(a.b[idx[u]], v);
        y[idx[u]] = v;
        if (MODE == SPMM_RESID_CYCLE) nacc += abs2(v);
      }
    }
  }
  if (MODE == SPMM_RESID_CYCLE) {
    __shared__ double s_n[kThreads];
    __shared__ double s_tot[8];
    s_n[threadIdx.x] = lane_ok ? nacc : 0.0;
    __syncthreads();
    if (threadIdx.x < R) {
      double t = 0.0;
      for (int w = 0; w < kWarps; ++w)
        for (int gq = 0; gq < GPW; ++gq) t += s_n[w * 32 + gq * R + threadIdx.x];
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
        fin_cycle(a.st, s_tot);
      }
      if (threadIdx.x == 0) *a.st.ticket = 0u;
    }
  }
}

// ----------------------------------------------------------------------------
// Kernel 2: block dot of classical Gram-Schmidt
//   h[i][c] = S[i][c] * sum_rows conj(V_i[row,c]) * w[row,c],  i = 0..j
//   (optionally ||w_c||^2), w = V_{j+1}.  Deterministic two-level reduction.
// ----------------------------------------------------------------------------
struct OrthArgs {
  long long n;
  const void* V;     // basis base (raw, unnormalised blocks)
  const void* Z;     // FGMRES Z base (x-update)
  void* x;           // solution (x-update)
  const void* dinv;  // Jacobi (x-update, GMRES form)
  long long stride;
  GState st;
};

template <typename XT, int R, bool PASS1>
__global__ void __launch_bounds__(kThreads) k_dot(OrthArgs a) {
  constexpr int GPW = 32 / R;
  constexpr int U = (R <= 2) ? 8 : 4;
  extern __shared__ double smem_d[];
  if (*a.st.any_active == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const int j = *a.st.j;
  const int J = j + 1;
  const XT* V = reinterpret_cast<const XT*>(a.V);
  const XT* w = V + (long long)J * a.stride;
  XT* s_acc = reinterpret_cast<XT*>(smem_d);          // [J][kWarps][R]
  double* s_w2 = reinterpret_cast<double*>(s_acc + (size_t)J * kWarps * R);  // [kWarps][R]
  for (int o = threadIdx.x; o < J * kWarps * R; o += kThreads) s_acc[o] = zero<XT>();
  if (PASS1) for (int o = threadIdx.x; o < kWarps * R; o += kThreads) s_w2[o] = 0.0;
  __syncthreads();

  const long long tile_rows = (long long)GPW * U;
  const long long ntiles = (a.n + tile_rows - 1) / tile_rows;
  double w2 = 0.0;
  for (long long t = (long long)blockIdx.x * kWarps + warp; t < ntiles;
       t += (long long)gridDim.x * kWarps) {
    XT wv[U];
    long long idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long row = t * tile_rows + u * GPW + grp;
      bool ok = lane_ok && row < a.n;
      idx[u] = ok ? row * R + c : -1;
      wv[u] = ok ? w[idx[u]] : zero<XT>();
      if (PASS1) w2 += abs2(wv[u]);
    }
    int i = 0;
    for (; i + 1 < J; i += 2) {
      const XT* v0 = V + (long long)i * a.stride;
      const XT* v1 = v0 + a.stride;
      XT p0 = zero<XT>(), p1 = zero<XT>();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (idx[u] >= 0) {
          p0 = cfma(v0[idx[u]], wv[u], p0);
          p1 = cfma(v1[idx[u]], wv[u], p1);
        }
      }
      p0 = group_reduce<R>(p0, grp);
      p1 = group_reduce<R>(p1, grp);
      if (grp == 0) {
        XT* s0 = s_acc + ((size_t)i * kWarps + warp) * R + c;
        *s0 = add(*s0, p0);
        XT* s1 = s0 + kWarps * R;
        *s1 = add(*s1, p1);
      }
    }
    if (i < J) {
      const XT* v0 = V + (long long)i * a.stride;
      XT p0 = zero<XT>();
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (idx[u] >= 0) p0 = cfma(v0[idx[u]], wv[u], p0);
      p0 = group_reduce<R>(p0, grp);
      if (grp == 0) {
        XT* s0 = s_acc + ((size_t)i * kWarps + warp) * R + c;
        *s0 = add(*s0, p0);
      }
    }
  }
  if (PASS1) {
    w2 = group_reduce<R>(w2, grp);
    if (grp == 0 && lane_ok) s_w2[warp * R + c] = w2;
  }
  __syncthreads();
  // block partial: [J*R complex][R doubles]
  double* part = a.st.part + (size_t)blockIdx.x * a.st.pstride;
  for (int o = threadIdx.x; o < J * R; o += kThreads) {
    int ii = o / R, cc = o - ii * R;
    XT t = zero<XT>();
    for (int wq = 0; wq < kWarps; ++wq) t = add(t, s_acc[((size_t)ii * kWarps + wq) * R + cc]);
    double2 tc = to_c(t);
    part[2 * o] = tc.x;
    part[2 * o + 1] = tc.y;
  }
  if (PASS1 && threadIdx.x < R) {
    double t = 0.0;
    for (int wq = 0; wq < kWarps; ++wq) t += s_w2[wq * R + threadIdx.x];
    part[2 * (a.st.m + 1) * R + threadIdx.x] = t;
  }
  if (a.st.rsum && last_block(a.st.ticket)) {
    // this rank's sums, unscaled; k_dist_fin scales the all-reduced values
    for (int o = threadIdx.x; o < J * R; o += kThreads) {
      double sx = 0.0, sy = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) {
        const double* pb = a.st.part + (size_t)b * a.st.pstride;
        sx += __ldcg(pb + 2 * o);
        sy += __ldcg(pb + 2 * o + 1);
      }
      a.st.rsum[2 * o] = sx;
      a.st.rsum[2 * o + 1] = sy;
    }
    if (PASS1 && threadIdx.x < R) {
      double t = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b)
        t += __ldcg(a.st.part + (size_t)b * a.st.pstride + 2 * (a.st.m + 1) * R + threadIdx.x);
      a.st.rsum[2 * (a.st.m + 1) * R + threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) *a.st.ticket = 0u;
  } else if (!a.st.rsum && last_block(a.st.ticket)) {
    double2* hout = PASS1 ? a.st.h : a.st.h2;
    for (int o = threadIdx.x; o < J * R; o += kThreads) {
      double sx = 0.0, sy = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) {
        const double* pb = a.st.part + (size_t)b * a.st.pstride;
        sx += __ldcg(pb + 2 * o);
        sy += __ldcg(pb + 2 * o + 1);
      }
      double s = a.st.S[o];   // S[i*R + c] with o = i*R + c
      hout[o] = s == 0.0 ? make_double2(0.0, 0.0) : make_double2(s * sx, s * sy);
    }
    if (PASS1 && threadIdx.x < R) {
      double t = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b)
        t += __ldcg(a.st.part + (size_t)b * a.st.pstride + 2 * (a.st.m + 1) * R + threadIdx.x);
      a.st.wpre2[threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) *a.st.ticket = 0u;
  }
}

// ----------------------------------------------------------------------------
// Kernel 3: block update
//   ORTH1: w -= sum_i V_i * (S_i h_i)
//   ORTH2: w -= sum_i V_i * (S_i h2_i), ||w_c||^2 -> fin_givens
//   XUPD : x += D^-1 sum_i V_i ycoef_i   (GMRES form)
//   XUPDF: x += sum_i Z_i ycoef_i        (FGMRES form)
// ----------------------------------------------------------------------------
enum UpdMode { UPD_ORTH1 = 0, UPD_ORTH2 = 1, UPD_X = 2, UPD_XF = 3 };

template <typename XT, int R, int MODE>
__global__ void __launch_bounds__(kThreads) k_update(OrthArgs a) {
  constexpr int GPW = 32 / R;
  constexpr int U = (R <= 2) ? 8 : 4;
  constexpr bool ORTH = (MODE == UPD_ORTH1 || MODE == UPD_ORTH2);
  extern __shared__ double smem_d[];
  if (ORTH && *a.st.any_active == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  int J;
  const XT* B;
  XT* tgt;
  if (ORTH) {
    J = *a.st.j + 1;
    B = reinterpret_cast<const XT*>(a.V);
    tgt = const_cast<XT*>(B) + (long long)J * a.stride;
  } else {
    J = *a.st.jx;
    B = reinterpret_cast<const XT*>(MODE == UPD_XF ? a.Z : a.V);
    tgt = reinterpret_cast<XT*>(a.x);
  }
  if (J == 0) return;
  XT* s_coef = reinterpret_cast<XT*>(smem_d);  // [J][R]
  for (int o = threadIdx.x; o < J * R; o += kThreads) {
    double2 cf;
    if (MODE == UPD_ORTH1) cf = a.st.h[o];
    else if (MODE == UPD_ORTH2) cf = a.st.h2[o];
    else cf = a.st.ycoef[o];
    if (ORTH) {
      double s = a.st.S[o];
      cf = s == 0.0 ? make_double2(0.0, 0.0) : make_double2(s * cf.x, s * cf.y);
    }
    s_coef[o] = from_c<XT>(cf);
  }
  __syncthreads();
  const XT* dinv = reinterpret_cast<const XT*>(a.dinv);
  const long long tile_rows = (long long)GPW * U;
  const long long ntiles = (a.n + tile_rows - 1) / tile_rows;
  double n2 = 0.0;
  for (long long t = (long long)blockIdx.x * kWarps + warp; t < ntiles;
       t += (long long)gridDim.x * kWarps) {
    XT acc[U];
    long long idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long row = t * tile_rows + u * GPW + grp;
      idx[u] = (lane_ok && row < a.n) ? row * R + c : -1;
      acc[u] = zero<XT>();
    }
    for (int i = 0; i < J; ++i) {
      const XT* bi = B + (long long)i * a.stride;
      const XT cf = s_coef[i * R + c];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (idx[u] >= 0) acc[u] = fma_(bi[idx[u]], cf, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (idx[u] < 0) continue;
      XT v = tgt[idx[u]];
      if (ORTH) {
        v = sub(v, acc[u]);
        if (MODE == UPD_ORTH2) n2 += abs2(v);
      } else if (MODE == UPD_X) {
        v = fma_(dinv[idx[u] / R], acc[u], v);
      } else {
        v = add(v, acc[u]);
      }
      tgt[idx[u]] = v;
    }
  }
  if (MODE == UPD_ORTH2) {
    __shared__ double s_n[kWarps * 8];
    __shared__ double s_tot[8];
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
}

// ----------------------------------------------------------------------------
// Row-partitioned solves.  Every reduction of the Arnoldi
// step is a rank-local sum (above, into st.rsum), an all-reduce over the ranks
// (NCCL, or the in-process group sum below), then this finisher, replicated on
// every rank so the Hessenberg, Givens and masks stay identical everywhere.
// ----------------------------------------------------------------------------
enum DistFin { FIN_DOT1 = 0, FIN_DOT2 = 1, FIN_GIVENS = 2, FIN_CYCLE = 3 };

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_dist_fin(GState st) {
  // inactive steps after the stop: the reducing kernels returned early and rsum
  // holds stale sums; nothing to finish (the cycle-end residual always runs)
  if (MODE != FIN_CYCLE && *st.any_active == 0) return;
  const int R = st.R;
  if (MODE == FIN_DOT1 || MODE == FIN_DOT2) {
    const int J = *st.j + 1;
    double2* hout = MODE == FIN_DOT1 ? st.h : st.h2;
    for (int o = threadIdx.x; o < J * R; o += kThreads) {
      const double s = st.S[o];
      hout[o] = s == 0.0 ? make_double2(0.0, 0.0)
                         : make_double2(s * st.rsum[2 * o], s * st.rsum[2 * o + 1]);
    }
    if (MODE == FIN_DOT1 && threadIdx.x < R) st.wpre2[threadIdx.x] = st.rsum[2 * (st.m + 1) * R + threadIdx.x];
  } else {
    __shared__ double s_tot[8];
    if (threadIdx.x < R) s_tot[threadIdx.x] = st.rsum[threadIdx.x];
    __syncthreads();
    if (MODE == FIN_GIVENS) fin_givens(st, s_tot);
    else fin_cycle(st, s_tot);
  }
}

// Sum `count` doubles over the P rank buffers of an in-process rank group (rank
// order, the same on every rank) and write the result back to every buffer.
static __global__ void k_group_sum(double* const* bufs, int P, int count) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int p = 0; p < P; ++p) t += bufs[p][i];
    for (int p = 0; p < P; ++p) bufs[p][i] = t;
  }
}

// Halo send buffer: rows `rows[0..count)` of an (n x wd doubles) block, packed.
static __global__ void k_halo_pack(const double* __restrict__ src, int wd, const int* __restrict__ rows,
                                   long long count, double* __restrict__ dst) {
  const long long total = count * wd;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / wd;
    const int k = (int)(e - i * wd);
    dst[e] = src[(long long)rows[i] * wd + k];
  }
}

// ----------------------------------------------------------------------------
// cycle end: back substitution of the rotated Hessenberg, x-update coefficients
// ----------------------------------------------------------------------------
static __global__ void k_trisolve(GState st, int flexible) {
  const int R = st.R, m = st.m;
  const int c = threadIdx.x;
  if (c < R) {
    int k = st.kdim[c];
    const double2* Hc = st.H + (size_t)c * m * (m + 1);
    const double2* gv = st.g + (size_t)c * (m + 1);
    for (int i = k - 1; i >= 0; --i) {
      double2 acc = gv[i];
      for (int l = i + 1; l < k; ++l) acc = sub(acc, mul(Hc[(size_t)l * (m + 1) + i], st.ycoef[l * R + c]));
      st.ycoef[i * R + c] = cdiv(acc, Hc[(size_t)i * (m + 1) + i]);
    }
    for (int i = 0; i < k; ++i) {
      if (!flexible) {
        double s = st.S[i * R + c];
        double2 y = st.ycoef[i * R + c];
        st.ycoef[i * R + c] = s == 0.0 ? make_double2(0.0, 0.0) : make_double2(s * y.x, s * y.y);
      }
    }
    for (int i = k; i < m; ++i) st.ycoef[i * R + c] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int jx = 0;
    for (int cc = 0; cc < R; ++cc) jx = max(jx, st.kdim[cc]);
    *st.jx = jx;
  }
}

// solve start: counters and flags
static __global__ void k_init(GState st) {
  if (threadIdx.x < st.R) {
    st.iters[threadIdx.x] = 0;
    st.done[threadIdx.x] = 0;
    st.active[threadIdx.x] = 0;
    st.kdim[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) {
    *st.j = 0;
    *st.any_active = 0;
    *st.jx = 0;
    *st.ticket = 0u;
    *st.stepseq = 0ull;
    *st.cycleseq = 0ull;
  }
}

// ----------------------------------------------------------------------------
// Gram matrix G = X^H Y (R x R), deterministic; result written to out[R*R]
// (complex) by the last block.
// ----------------------------------------------------------------------------
template <typename XT, int R>
__global__ void __launch_bounds__(kThreads) k_gram(long long n, const XT* X, const XT* Y,
                                                   double* part, unsigned* ticket, double2* out) {
  __shared__ double2 s_w[kWarps][R * R];
  XT acc[R * R];
#pragma unroll
  for (int q = 0; q < R * R; ++q) acc[q] = zero<XT>();
  for (long long row = (long long)blockIdx.x * kThreads + threadIdx.x; row < n;
       row += (long long)gridDim.x * kThreads) {
    XT xr[R], yr[R];
#pragma unroll
    for (int q = 0; q < R; ++q) { xr[q] = X[row * R + q]; yr[q] = Y[row * R + q]; }
#pragma unroll
    for (int p = 0; p < R; ++p)
#pragma unroll
      for (int q = 0; q < R; ++q) acc[p * R + q] = cfma(xr[p], yr[q], acc[p * R + q]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < R * R; ++q) {
    XT v = acc[q];
    for (int s = 16; s > 0; s >>= 1) v = add(v, shfl_down(v, s));
    if (lane == 0) s_w[warp][q] = to_c(v);
  }
  __syncthreads();
  if (threadIdx.x < R * R) {
    double2 t = make_double2(0.0, 0.0);
    for (int wq = 0; wq < kWarps; ++wq) t = add(t, s_w[wq][threadIdx.x]);
    part[(size_t)blockIdx.x * 2 * R * R + 2 * threadIdx.x] = t.x;
    part[(size_t)blockIdx.x * 2 * R * R + 2 * threadIdx.x + 1] = t.y;
  }
  if (last_block(ticket)) {
    if (threadIdx.x < R * R) {
      double sx = 0.0, sy = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) {
        sx += __ldcg(part + (size_t)b * 2 * R * R + 2 * threadIdx.x);
        sy += __ldcg(part + (size_t)b * 2 * R * R + 2 * threadIdx.x + 1);
      }
      out[threadIdx.x] = make_double2(sx, sy);
    }
    __syncthreads();
    if (threadIdx.x == 0) *ticket = 0u;
  }
}

// y += a*x over n*R elements
template <typename XT>
__global__ void k_axpy(long long count, double2 a, const XT* x, XT* y) {
  const XT av = from_c<XT>(a);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = fma_(av, x[i], y[i]);
}

// Jacobi: dinv[row] = 1 / (diag(A)[row] + sigma * massdiag)   (complex); flags |d| < 1e-300
template <typename VT>
__global__ void k_jacobi(long long n, const int* rowptr, const int* colidx, const VT* vals,
                         double2 sigma, int sigma_identity, double2* dinv, int* breakdown) {
  for (long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (long long)gridDim.x * blockDim.x) {
    double2 d = make_double2(0.0, 0.0);
    for (int k = rowptr[row]; k < rowptr[row + 1]; ++k) {
      if (colidx[k] == row) { d = to_c(vals[k]); break; }
    }
    if (sigma_identity) d = add(d, sigma);
    if (hypot(d.x, d.y) < 1e-300) {
      atomicOr(breakdown, 1);
      dinv[row] = make_double2(0.0, 0.0);
    } else {
      dinv[row] = cdiv(make_double2(1.0, 0.0), d);
    }
  }
}

static __global__ void k_c2r(long long n, const double2* in, double* out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i].x;
}

}  // namespace sad
