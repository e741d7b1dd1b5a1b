// sad_bicg.cuh -- the reference's own inner solver on the device: right-
// preconditioned BiCGstab (krylov.py:82-157) with the drift-resume loop of
// bicgstab() (krylov.py:160-184), batched over the r columns of a block.
//
// Each column is an independent BiCGstab run; the columns advance in lock
// step through five kernels per iteration, every one of which ends in a
// last-block finisher that updates the column's scalars (rho, alpha, omega,
// beta, breakdown restarts, stopping) on the device:
//   PUPD  p = r + beta (p - omega v)            (p = r, rhat = r after a restart)
//   SPMM1 v = Op(D^-1 p),   denom = <rhat, v>   -> alpha, breakdown
//   SUPD  s = r - alpha v,  dx += alpha D^-1 p,  ||s|| -> it++, stop on ||s|| <= tol
//   SPMM2 t = Op(D^-1 s),   <t,t>, <t,s>        -> omega, breakdowns
//   RUPD  dx += omega D^-1 s, r = s - omega t,  ||r||, <rhat,r>, ||rhat|| -> rho,
//         stop on ||r|| <= tol, next rho_new / beta (the loop top)
// A "run" is one _bicgstab_column call; at the end of a run the solution is
// x += dx (the reference's xc = xc + dx) and the true residual b - Op x is
// recomputed; a column resumes from it while ||true|| > tol, budget remains
// and the previous run made progress (krylov.py:170-181).
// Flags and masks live in device memory; the host only stops issuing
// iterations once a host-mapped flag says no column is active.
#pragma once

#include "sad_kernels.cuh"

namespace sad {

constexpr double kBiTiny = 1e-290;   // krylov.py:79 _BREAKDOWN_TINY

struct BState {
  // per column [R]
  double2* rho;
  double2* alpha;
  double2* omega;
  double2* rho_new;
  double2* beta;
  double* scale;      // ||rhat|| ||r|| at the loop top
  double* nr2;        // ||r||^2 at the loop top
  double* tnorm;      // ||b - Op x|| after the last run
  long long* it;      // iterations of the column (all runs)
  long long* run_it;  // iterations of the current run
  int* active;        // current run still iterating
  int* ok;            // column iterating (set by the loop top, cleared at the run's end)
  int* skip;          // rest of this iteration skipped (denominator breakdown restart)
  int* fresh;         // next PUPD: rhat = r, p = r (after a restart)
  int* rmode;         // next RUPD: r = rhat = s (restart from s)
  int* restarted;
  int* inrun;         // column takes part in the current run
  int* any_active;
  unsigned* ticket;
  double* part;       // [blocks][pstride]
  unsigned long long* stepseq;
  unsigned long long* cycleseq;
  volatile long long* hflag;   // [0] stepseq [1] any_active [2] cycleseq [3] any resuming
  double tol;
  long long maxit;
  int R;
  int pstride;
};

struct BArgs {
  long long n;
  const int* rowptr;
  const int* colidx;
  const void* vals;
  double2 sigma;
  const void* dinv;
  const void* b;
  void *x, *dx, *r, *rhat, *p, *v, *s, *t;
  // general right preconditioner (incomplete factorisations, sad_precond_host.cuh):
  // phat = M^-1 p and shat = M^-1 s computed between the kernels; nullptr = the
  // fused Jacobi scaling by dinv
  const void* phat;
  const void* shat;
  BState st;
};

enum BiVec { BI_START = 0, BI_PUPD = 1, BI_SUPD = 2, BI_RUPD = 3, BI_XUPD = 4 };
enum BiSpmm { BI_SPMM_P = 0, BI_SPMM_S = 1, BI_RESID = 2 };

// ---- finishers ----------------------------------------------------------------
__device__ __forceinline__ double cabs2_(double2 a) { return hypot(a.x, a.y); }

// end of a run for column c (the run's `return x, it` or `break`)
__device__ __forceinline__ void bi_end(const BState& st, int c) {
  st.active[c] = 0;
  st.ok[c] = 0;
}

// loop top (krylov.py:94-110): the iteration cap, rho_new and its breakdown
// restart, beta.  rho_new/nrhat2/nr2 describe the current r and rhat.
static __device__ void bi_top(const BState& st, int c, double2 rho_new, double nrhat2, double nr2) {
  if (st.run_it[c] >= st.maxit - (st.it[c] - st.run_it[c])) { bi_end(st, c); return; }
  double scale = sqrt(nrhat2) * sqrt(nr2);
  if (cabs2_(rho_new) <= kBiTiny * fmax(scale, 1.0)) {
    if (st.restarted[c]) { bi_end(st, c); return; }
    // rhat = r, rho = alpha = omega = 1, v = p = 0, then the loop top again
    st.fresh[c] = 1;
    st.restarted[c] = 1;
    st.rho[c] = st.alpha[c] = st.omega[c] = make_double2(1.0, 0.0);
    rho_new = make_double2(nr2, 0.0);
    scale = nr2;
    if (cabs2_(rho_new) <= kBiTiny * fmax(scale, 1.0)) { bi_end(st, c); return; }
  }
  st.rho_new[c] = rho_new;
  st.scale[c] = scale;
  st.nr2[c] = nr2;
  st.beta[c] = mul(cdiv(rho_new, st.rho[c]), cdiv(st.alpha[c], st.omega[c]));
  st.ok[c] = 1;
}

// tot layout per kernel: [q][R] doubles, complex quantities as two entries
static __device__ void bi_finish_vec(const BState& st, int K, const double* tot) {
  const int R = st.R;
  const int c = threadIdx.x;
  if (c < R) {
    if (K == BI_START) {
      if (st.inrun[c]) {
        const double nr2 = tot[c];
        st.run_it[c] = 0;
        st.restarted[c] = 0;
        st.fresh[c] = 1;          // v = p = 0: the first PUPD sets p = r
        st.rmode[c] = 0;
        st.rho[c] = st.alpha[c] = st.omega[c] = make_double2(1.0, 0.0);
        if (sqrt(nr2) <= st.tol) {          // krylov.py:87-88
          bi_end(st, c);
        } else {
          st.active[c] = 1;
          bi_top(st, c, make_double2(tot[3 * R + c], tot[4 * R + c]), tot[R + c], nr2);
        }
      } else {
        bi_end(st, c);
      }
    } else if (K == BI_SUPD) {
      if (st.ok[c] && !st.skip[c]) {
        st.it[c] += 1;
        st.run_it[c] += 1;
        if (sqrt(tot[c]) <= st.tol) bi_end(st, c);
      }
    } else if (K == BI_RUPD) {
      if (st.ok[c] && !st.skip[c]) {
        const double nr2 = tot[c];
        const double2 rn = make_double2(tot[3 * R + c], tot[4 * R + c]);
        if (st.rmode[c]) {
          // restart from s (krylov.py:131-150): `continue` to the loop top
          st.rmode[c] = 0;
          st.fresh[c] = 1;
          bi_top(st, c, rn, tot[R + c], nr2);
        } else {
          st.rho[c] = st.rho_new[c];
          if (sqrt(nr2) <= st.tol) bi_end(st, c);
          else bi_top(st, c, rn, tot[R + c], nr2);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && K == BI_RUPD) {
    int any = 0;
    for (int cc = 0; cc < R; ++cc) any |= st.active[cc];
    *st.any_active = any;
    unsigned long long sq = ++(*st.stepseq);
    st.hflag[1] = any;
    __threadfence_system();
    st.hflag[0] = (long long)sq;
  }
  if (threadIdx.x == 0 && K == BI_START) {
    int any = 0;
    for (int cc = 0; cc < R; ++cc) any |= st.active[cc];
    *st.any_active = any;
  }
}

static __device__ void bi_finish_spmm(const BState& st, int K, const double* tot) {
  const int R = st.R;
  const int c = threadIdx.x;
  if (c < R) {
    if (K == BI_SPMM_P) {
      st.fresh[c] = 0;              // PUPD has consumed it
      st.skip[c] = 0;
      if (st.ok[c]) {
        const double2 denom = make_double2(tot[c], tot[R + c]);
        if (cabs2_(denom) <= kBiTiny * fmax(st.scale[c], 1.0)) {
          if (st.restarted[c]) {
            bi_end(st, c);
          } else {
            // rhat = r, scalars reset, `continue` to the loop top with rhat = r
            st.restarted[c] = 1;
            st.rho[c] = st.alpha[c] = st.omega[c] = make_double2(1.0, 0.0);
            const double nr2 = st.nr2[c];
            bi_top(st, c, make_double2(nr2, 0.0), nr2, nr2);
            st.skip[c] = 1;                     // SUPD..RUPD of this iteration
            st.fresh[c] = st.active[c];         // next PUPD: rhat = r, p = r
          }
        } else {
          st.alpha[c] = cdiv(st.rho_new[c], denom);
        }
      }
    } else if (K == BI_SPMM_S) {
      if (st.ok[c] && !st.skip[c]) {
        const double tt = tot[c];
        const double2 ts = make_double2(tot[R + c], tot[2 * R + c]);
        bool restart = tt <= kBiTiny;
        if (!restart) {
          st.omega[c] = make_double2(ts.x / tt, ts.y / tt);
          restart = cabs2_(st.omega[c]) <= kBiTiny;
        }
        if (restart) {
          if (st.restarted[c]) {
            bi_end(st, c);
          } else {
            st.restarted[c] = 1;
            st.rho[c] = st.alpha[c] = st.omega[c] = make_double2(1.0, 0.0);
            st.rmode[c] = 1;
          }
        }
      }
    } else {  // BI_RESID: end of a run, decide the resume (krylov.py:170-181)
      const double tn = sqrt(tot[c]);
      st.tnorm[c] = tn;
      const bool resume = st.inrun[c] && tn > st.tol && st.it[c] < st.maxit && st.run_it[c] > 0;
      st.inrun[c] = resume ? 1 : 0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && K == BI_RESID) {
    int any = 0;
    for (int cc = 0; cc < R; ++cc) any |= st.inrun[cc];
    unsigned long long cs = ++(*st.cycleseq);
    st.hflag[3] = any;
    __threadfence_system();
    st.hflag[2] = (long long)cs;
  }
}

// ---- per-block partial sums -> last block ------------------------------------
// NQ doubles per column; partial layout [block][NQ][R].  Returns true in the
// last block to arrive, with the totals in tot_s[NQ * R] (block order: fixed).
template <int R, int NQ>
__device__ __forceinline__ bool part_reduce(double* part, int pstride, unsigned* ticket,
                                            const double (&q)[NQ], int grp, int c, bool lane_ok,
                                            double* tot_s) {
  __shared__ double s_q[kWarps][NQ][8];
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NQ; ++k) {
    double v = group_reduce<R>(q[k], grp);
    if (grp == 0 && lane_ok) s_q[warp][k][c] = v;
  }
  __syncthreads();
  if (threadIdx.x < NQ * R) {
    const int k = threadIdx.x / R, cc = threadIdx.x - k * R;
    double t = 0.0;
    for (int w = 0; w < kWarps; ++w) t += s_q[w][k][cc];
    part[(size_t)blockIdx.x * pstride + threadIdx.x] = t;
  }
  if (!last_block(ticket)) return false;
  // all outputs together, 8 at a time: each thread sums its strided blocks for
  // 8 outputs (independent loads in flight), then one shared-memory tree for the
  // 8 (fixed order: deterministic)
  __shared__ double s_red[8][kThreads];
  for (int o0 = 0; o0 < NQ * R; o0 += 8) {
    const int no = min(8, NQ * R - o0);
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kThreads) {
      const double* pb = part + (size_t)b * pstride + o0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < no) acc[k] += __ldcg(pb + k);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s_red[k][threadIdx.x] = acc[k];
    __syncthreads();
    for (int sh = kThreads / 2; sh > 0; sh >>= 1) {
      if (threadIdx.x < sh) {
#pragma unroll
        for (int k = 0; k < 8; ++k) s_red[k][threadIdx.x] += s_red[k][threadIdx.x + sh];
      }
      __syncthreads();
    }
    if (threadIdx.x < no) tot_s[o0 + threadIdx.x] = s_red[threadIdx.x][0];
    __syncthreads();
  }
  __syncthreads();
  return true;
}

template <int R, int NQ>
__device__ __forceinline__ bool bi_reduce(const BState& st, const double (&q)[NQ], int grp, int c,
                                          bool lane_ok, double* tot_s) {
  return part_reduce<R, NQ>(st.part, st.pstride, st.ticket, q, grp, c, lane_ok, tot_s);
}

// ---- elementwise kernels ------------------------------------------------------
template <typename XT, int R, int K>
__global__ void __launch_bounds__(kThreads) k_bi_vec(BArgs a) {
  constexpr int GPW = 32 / R;
  constexpr int NQ = (K == BI_START || K == BI_RUPD) ? 5 : (K == BI_SUPD ? 1 : 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const BState& st = a.st;
  const XT* dinv = reinterpret_cast<const XT*>(a.dinv);
  XT* x = reinterpret_cast<XT*>(a.x);
  XT* dx = reinterpret_cast<XT*>(a.dx);
  XT* r = reinterpret_cast<XT*>(a.r);
  XT* rhat = reinterpret_cast<XT*>(a.rhat);
  XT* p = reinterpret_cast<XT*>(a.p);
  const XT* v = reinterpret_cast<const XT*>(a.v);
  XT* s = reinterpret_cast<XT*>(a.s);
  const XT* t = reinterpret_cast<const XT*>(a.t);
  const XT* phat = reinterpret_cast<const XT*>(a.phat);
  const XT* shat = reinterpret_cast<const XT*>(a.shat);
  // column flags and coefficients (read once)
  int on = 0, fr = 0, rm = 0;
  XT cb = zero<XT>(), co = zero<XT>(), ca = zero<XT>();
  if (lane_ok) {
    if (K == BI_START || K == BI_XUPD) on = st.inrun[c];
    else if (K == BI_PUPD) on = st.ok[c];
    else on = st.ok[c] && !st.skip[c];
    fr = st.fresh[c];
    rm = st.rmode[c];
    cb = from_c<XT>(st.beta[c]);
    co = from_c<XT>(st.omega[c]);
    ca = from_c<XT>(st.alpha[c]);
  }
  double q[NQ > 0 ? NQ : 1];
#pragma unroll
  for (int k = 0; k < (NQ > 0 ? NQ : 1); ++k) q[k] = 0.0;
  (void)q;
  const long long rows_per_iter = (long long)gridDim.x * kWarps * GPW;
  if (lane_ok && on) {
    for (long long row = ((long long)blockIdx.x * kWarps + warp) * GPW + grp; row < a.n;
         row += rows_per_iter) {
      const long long e = row * R + c;
      if (K == BI_START) {
        const XT rv = r[e];
        rhat[e] = rv;
        dx[e] = zero<XT>();
        const double n2 = abs2(rv);
        q[0] += n2;
        q[1] += n2;
        const double2 rr = to_c(cfma(rv, rv, zero<XT>()));
        q[3] += rr.x;
        q[4] += rr.y;
      } else if (K == BI_PUPD) {
        const XT rv = r[e];
        if (fr) {
          rhat[e] = rv;
          p[e] = rv;
        } else {
          // p = r + beta * (p - omega * v)
          const XT pv = p[e];
          const XT inner = sub(pv, mul(co, v[e]));
          p[e] = add(rv, mul(cb, inner));
        }
      } else if (K == BI_SUPD) {
        const XT sv = sub(r[e], mul(ca, v[e]));
        s[e] = sv;
        const XT ph = phat ? phat[e] : mul(dinv[row], p[e]);
        dx[e] = add(dx[e], mul(ca, ph));
        q[0] += abs2(sv);
      } else if (K == BI_RUPD) {
        const XT sv = s[e];
        XT rv, rh;
        if (rm) {
          rv = sv;
          rh = sv;
          r[e] = rv;
          rhat[e] = rh;
        } else {
          const XT sh = shat ? shat[e] : mul(dinv[row], sv);
          dx[e] = add(dx[e], mul(co, sh));
          rv = sub(sv, mul(co, t[e]));
          r[e] = rv;
          rh = rhat[e];
        }
        q[0] += abs2(rv);
        q[1] += abs2(rh);
        const double2 d = to_c(cfma(rh, rv, zero<XT>()));
        q[3] += d.x;
        q[4] += d.y;
      } else {  // BI_XUPD: x = x + dx
        x[e] = add(x[e], dx[e]);
      }
    }
  }
  if constexpr (NQ > 0) {
    __shared__ double tot_s[5 * 8];
    if (bi_reduce<R, NQ>(st, q, grp, c, lane_ok, tot_s)) {
      bi_finish_vec(st, K, tot_s);
      __syncthreads();
      if (threadIdx.x == 0) *st.ticket = 0u;
    }
  }
}

// ---- SpMM kernels with fused dots ------------------------------------------------
template <typename XT, typename VT, int R, int K, bool SIGMA>
__global__ void __launch_bounds__(kThreads) k_bi_spmm(BArgs a) {
  constexpr int GPW = 32 / R;
  constexpr int NQ = (K == BI_SPMM_P) ? 2 : (K == BI_SPMM_S ? 3 : 1);
  constexpr bool PRE = (K != BI_RESID);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const BState& st = a.st;
  const VT* vals = reinterpret_cast<const VT*>(a.vals);
  const XT* dinv = reinterpret_cast<const XT*>(a.dinv);
  // with a general preconditioner the operator is applied to phat / shat (its dinv is 1)
  const XT* in = reinterpret_cast<const XT*>(
      K == BI_SPMM_P ? (a.phat ? a.phat : a.p) : (K == BI_SPMM_S ? (a.shat ? a.shat : a.s) : a.x));
  XT* out = reinterpret_cast<XT*>(K == BI_SPMM_P ? a.v : (K == BI_SPMM_S ? a.t : a.r));
  const XT* other = reinterpret_cast<const XT*>(K == BI_SPMM_P ? a.rhat : (K == BI_SPMM_S ? a.s : a.b));
  bool on = lane_ok;
  if (K == BI_SPMM_P && lane_ok) on = st.ok[c] != 0;
  if (K == BI_SPMM_S && lane_ok) on = st.ok[c] && !st.skip[c];
  double q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) q[k] = 0.0;
  const long long rows_per_iter = (long long)gridDim.x * kWarps * GPW;
  constexpr int U = 2;
  // the whole group walks the rows (lanes of inactive columns still gather so
  // the group's loads stay converged; their results are discarded)
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
      spmm_rows<XT, VT, PRE, SIGMA, R, U>(a.rowptr, a.colidx, vals, dinv, a.sigma, in, idx, c,
                                          acc, xi);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (idx[u] < 0 || !on) continue;
        XT y = acc[u];
        if (K == BI_RESID) y = sub(other[idx[u]], y);
        out[idx[u]] = y;
        if (K == BI_SPMM_P) {
          const double2 d = to_c(cfma(other[idx[u]], y, zero<XT>()));   // <rhat, v>
          q[0] += d.x;
          q[1] += d.y;
        } else if (K == BI_SPMM_S) {
          q[0] += abs2(y);                                               // <t, t>
          const double2 d = to_c(cfma(y, other[idx[u]], zero<XT>()));    // <t, s>
          q[1] += d.x;
          q[2] += d.y;
        } else {
          q[0] += abs2(y);
        }
      }
    }
  }
  __shared__ double tot_s[5 * 8];
  if (bi_reduce<R, NQ>(st, q, grp, c, lane_ok, tot_s)) {
    bi_finish_spmm(st, K, tot_s);
    __syncthreads();
    if (threadIdx.x == 0) *st.ticket = 0u;
  }
}

}  // namespace sad
