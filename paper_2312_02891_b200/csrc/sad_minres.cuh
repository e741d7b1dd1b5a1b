// sad_minres.cuh -- the reference's inner solver for Hermitian sides on the
// device: split-preconditioned MINRES (Paige-Saunders, krylov.py:187-268) per
// column, batched over the r columns of a block (krylov.py:271-287).
//
// SolverBinding dispatches to MINRES when the side is symmetric, the shift is
// real and the preconditioner has an SPD split (adi.py:468-488); for Jacobi the
// split is |dinv| (precond.py:242-256), for "none" the identity.
//
// The columns advance in lock step; one iteration is four kernels, the first
// two ending in a last-block finisher that updates the column's scalars:
//   SPMM   v = y / beta (written), y' = Op v - (beta/oldb) r1,  <v, y'>  -> alfa, it++
//   YUPD   r1 <- y' - (alfa/beta) r2 (the new r2, roles swapped on the host),
//          y = |dinv| r2, <r2, y> -> beta and the Givens recurrence (delta,
//          gbar, epsln, dbar, gamma, cs, sn, phi, phibar), the check trigger
//          (phibar <= check_at) and the stop flags
//   WUPD   w' = (v - oldeps w2 - delta w) / gamma, w2 <- w, w <- w', x += phi w'
//   CHECK  only if some column triggered: ||b - Op x|| -> converged / stop /
//          check_at = min(check_at, tol phibar / (2 ||r||))
// so the operation order per element is the reference's.  The host only stops
// issuing iterations once a host-mapped flag says no column is active.
#pragma once

#include "sad_bicg.cuh"

namespace sad {

struct MState {
  // per column [R]
  double* beta;
  double* oldb;
  double* dbar;
  double* epsln;
  double* phibar;
  double* cs;
  double* sn;
  double* check_at;
  double* alfa;
  double* c_oldeps;   // WUPD coefficients of the current iteration
  double* c_delta;
  double* c_gamma;
  double* c_phi;
  double* tnorm;      // ||b - Op x|| at the end
  long long* it;
  int* active;        // column iterating
  int* upd;           // WUPD applies this iteration
  int* chk;           // CHECK applies this iteration
  int* stop;          // stop after this iteration unless the check ends it first
  int* any_chk;
  int* err;           // beta1^2 <= 0 (krylov.py:203-205)
  unsigned* ticket;
  double* part;
  unsigned long long* stepseq;
  volatile long long* hflag;   // [0] stepseq [1] any_active
  double tol;
  long long maxit;
  int R;
  int pstride;
};

struct MArgs {
  long long n;
  const int* rowptr;
  const int* colidx;
  const void* vals;
  double2 sigma;
  const void* dinv;   // Jacobi dinv (XT); |dinv| is the SPD split
  const void* b;
  void *x, *r1, *r2, *y, *t, *v, *w, *w2;
  // 0: y = |dinv| r2 fused (none / Jacobi).  Cholesky kinds (apply_spd,
  // precond.py:242-256) split START and YUPD around the triangular solves:
  // 1 = write the vectors and y = r2 (no reduction), 2 = the dots on the solved y
  // and the finisher
  int pmode;
  MState st;
};

enum MrVec { MR_START = 0, MR_YUPD = 1, MR_WUPD = 2 };
// distinct from MrVec: mr_finish dispatches on one integer for both kinds
enum MrSpmm { MR_SPMM = 10, MR_CHECK = 11, MR_RESID = 12 };

constexpr double kMrTiny = 1e-300;

// numpy divides a complex array by a real scalar as a multiplication by the
// reciprocal (Smith's algorithm with a zero imaginary part): same here
__device__ __forceinline__ double sdiv(double a, double g) { return a * (1.0 / g); }
__device__ __forceinline__ double2 sdiv(double2 a, double g) {
  const double s = 1.0 / g;
  return make_double2(a.x * s, a.y * s);
}
__device__ __forceinline__ double pabs(double d) { return fabs(d); }
__device__ __forceinline__ double pabs(double2 d) { return hypot(d.x, d.y); }

// ---- finishers -----------------------------------------------------------------
static __device__ void mr_finish(const MState& st, int K, const double* tot) {
  const int R = st.R;
  const int c = threadIdx.x;
  if (c < R) {
    if (K == MR_START) {
      // krylov.py:192-221: ||b||, beta1, the recurrence start, check_at
      const double nb = sqrt(tot[c]);
      st.it[c] = 0;
      st.upd[c] = 0;
      st.chk[c] = 0;
      st.stop[c] = 0;
      st.active[c] = 0;
      if (!(nb <= st.tol)) {
        const double b1sq = tot[R + c];
        if (b1sq <= 0.0) {
          *st.err = 1;
          st.tnorm[c] = b1sq;
        } else {
          const double beta1 = sqrt(b1sq);
          st.oldb[c] = 0.0;
          st.beta[c] = beta1;
          st.dbar[c] = 0.0;
          st.epsln[c] = 0.0;
          st.phibar[c] = beta1;
          st.cs[c] = -1.0;
          st.sn[c] = 0.0;
          const double ratio = nb / beta1;
          st.check_at[c] = st.tol / fmax(ratio, kMrTiny);
          st.active[c] = st.maxit > 0 ? 1 : 0;
        }
      }
    } else if (K == MR_SPMM) {
      if (st.active[c]) {
        st.it[c] += 1;
        st.alfa[c] = tot[c];
      }
    } else if (K == MR_YUPD) {
      const int on = st.active[c];
      st.upd[c] = on;
      st.chk[c] = 0;
      if (on) {
        const double alfa = st.alfa[c];
        const double beta = sqrt(fmax(tot[c], 0.0));
        st.oldb[c] = st.beta[c];
        st.beta[c] = beta;
        const double cs = st.cs[c], sn = st.sn[c], dbar = st.dbar[c];
        const double oldeps = st.epsln[c];
        const double delta = cs * dbar + sn * alfa;
        const double gbar = sn * dbar - cs * alfa;
        st.epsln[c] = sn * beta;
        st.dbar[c] = -cs * beta;
        const double gamma = fmax(hypot(gbar, beta), kMrTiny);
        const double cs2 = gbar / gamma;
        const double sn2 = beta / gamma;
        const double phibar = st.phibar[c];
        const double phi = cs2 * phibar;
        const double phibar2 = sn2 * phibar;
        st.cs[c] = cs2;
        st.sn[c] = sn2;
        st.phibar[c] = phibar2;
        st.c_oldeps[c] = oldeps;
        st.c_delta[c] = delta;
        st.c_gamma[c] = gamma;
        st.c_phi[c] = phi;
        const int chk = phibar2 <= st.check_at[c];
        const int stop = (beta <= kMrTiny) || st.it[c] >= st.maxit;
        st.chk[c] = chk;
        st.stop[c] = stop;
        if (!chk && stop) st.active[c] = 0;
      }
    } else if (K == MR_CHECK) {
      if (st.chk[c]) {
        const double nr = sqrt(tot[c]);
        const double phibar = st.phibar[c];
        if (nr <= st.tol) {
          st.active[c] = 0;                      // return x, it
        } else if (phibar <= kMrTiny) {
          st.active[c] = 0;                      // break
        } else {
          st.check_at[c] = fmin(st.check_at[c], 0.5 * st.tol * phibar / nr);
          if (st.stop[c]) st.active[c] = 0;
        }
        st.chk[c] = 0;
      }
    } else {  // MR_RESID: _finalize (krylov.py:61-70)
      st.tnorm[c] = sqrt(tot[c]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && K == MR_YUPD) {
    int any = 0, anyc = 0;
    for (int cc = 0; cc < R; ++cc) {
      any |= st.active[cc];
      anyc |= st.chk[cc];
    }
    *st.any_chk = anyc;
    unsigned long long sq = ++(*st.stepseq);
    st.hflag[1] = any;
    __threadfence_system();
    st.hflag[0] = (long long)sq;
  }
}

// ---- elementwise kernels ------------------------------------------------------
template <typename XT, int R, int K>
__global__ void __launch_bounds__(kThreads) k_mr_vec(MArgs a) {
  constexpr int GPW = 32 / R;
  constexpr int NQ = (K == MR_START) ? 2 : (K == MR_YUPD ? 1 : 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const MState& st = a.st;
  const XT* dinv = reinterpret_cast<const XT*>(a.dinv);
  const XT* b = reinterpret_cast<const XT*>(a.b);
  XT* x = reinterpret_cast<XT*>(a.x);
  XT* r1 = reinterpret_cast<XT*>(a.r1);
  XT* r2 = reinterpret_cast<XT*>(a.r2);
  XT* y = reinterpret_cast<XT*>(a.y);
  const XT* t = reinterpret_cast<const XT*>(a.t);
  const XT* v = reinterpret_cast<const XT*>(a.v);
  XT* w = reinterpret_cast<XT*>(a.w);
  XT* w2 = reinterpret_cast<XT*>(a.w2);
  int on = 0;
  double cf = 0.0, ce = 0.0, cd = 0.0, cg = 1.0, cp = 0.0;
  if (lane_ok) {
    if (K == MR_START) on = 1;
    else if (K == MR_YUPD) on = st.active[c];
    else on = st.upd[c];
    if (K == MR_YUPD && on) cf = st.alfa[c] / st.beta[c];
    if (K == MR_WUPD && on) {
      ce = st.c_oldeps[c];
      cd = st.c_delta[c];
      cg = st.c_gamma[c];
      cp = st.c_phi[c];
    }
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
      if (K == MR_START) {
        // r1 = r2 = b, y = P r1, w = w2 = x = 0
        const XT bv = b[e];
        XT yv;
        if (a.pmode == 2) {
          yv = y[e];
        } else {
          r1[e] = bv;
          r2[e] = bv;
          yv = a.pmode == 1 ? bv : sscal(pabs(dinv[row]), bv);
          y[e] = yv;
          w[e] = zero<XT>();
          w2[e] = zero<XT>();
          x[e] = zero<XT>();
        }
        q[0] += abs2(bv);
        q[1] += to_c(cfma(bv, yv, zero<XT>())).x;   // Re <r1, y>
      } else if (K == MR_YUPD) {
        // y -= (alfa / beta) r2; r1 <- y (the new r2); y = P r2
        XT yv, py;
        if (a.pmode == 2) {
          yv = r1[e];
          py = y[e];
        } else {
          yv = sub(t[e], sscal(cf, r2[e]));
          r1[e] = yv;
          py = a.pmode == 1 ? yv : sscal(pabs(dinv[row]), yv);
          y[e] = py;
        }
        q[0] += to_c(cfma(yv, py, zero<XT>())).x;     // Re <r2, y>
      } else {  // MR_WUPD
        // w = (v - oldeps w1 - delta w2) / gamma with w1 = old w2, w2 = old w
        const XT wo = w[e];
        const XT num = sub(sub(v[e], sscal(ce, w2[e])), sscal(cd, wo));
        const XT wn = sdiv(num, cg);
        w2[e] = wo;
        w[e] = wn;
        x[e] = add(x[e], sscal(cp, wn));
      }
    }
  }
  if constexpr (NQ > 0) {
    if (a.pmode == 1) return;   // uniform: the dots follow the triangular solves
    __shared__ double tot_s[2 * 8];
    if (part_reduce<R, NQ>(st.part, st.pstride, st.ticket, q, grp, c, lane_ok, tot_s)) {
      mr_finish(st, K, tot_s);
      __syncthreads();
      if (threadIdx.x == 0) *st.ticket = 0u;
    }
  }
}

// ---- SpMM kernels ----------------------------------------------------------------
// MR_SPMM: v = y / beta for the own rows, y' = Op v - (beta / oldb) r1 (it >= 2),
//          <v, y'>.  The gathered neighbours are scaled exactly as v is.
// MR_CHECK / MR_RESID: b - Op x (CHECK: norms only, columns that triggered;
//          RESID: written to the residual block, every column).
template <typename XT, typename VT, int R, int K, bool SIGMA>
__global__ void __launch_bounds__(kThreads) k_mr_spmm(MArgs a) {
  constexpr int GPW = 32 / R;
  const MState& st = a.st;
  if (K == MR_CHECK) {
    if (__ldcg(st.any_chk) == 0) return;   // uniform across the grid
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const VT* vals = reinterpret_cast<const VT*>(a.vals);
  const XT* in = reinterpret_cast<const XT*>(K == MR_SPMM ? a.y : a.x);
  const XT* r1 = reinterpret_cast<const XT*>(a.r1);
  const XT* b = reinterpret_cast<const XT*>(a.b);
  XT* vout = reinterpret_cast<XT*>(a.v);
  XT* out = reinterpret_cast<XT*>(a.t);   // SPMM: y'; RESID: the residual block
  bool on = lane_ok;
  double sc = 1.0, cb = 0.0;
  bool sub_r1 = false;
  if (lane_ok) {
    if (K == MR_SPMM) {
      on = st.active[c] != 0;
      if (on) {
        const double be = st.beta[c];
        sc = 1.0 / be;
        sub_r1 = st.it[c] >= 1;                    // the coming iteration is it >= 2
        if (sub_r1) cb = be / st.oldb[c];
      }
    } else if (K == MR_CHECK) {
      on = st.chk[c] != 0;
    }
  }
  double q = 0.0;
  const long long rows_per_iter = (long long)gridDim.x * kWarps * GPW;
  constexpr int U = 2;
  if (lane_ok) {
    for (long long row0 = ((long long)blockIdx.x * kWarps + warp) * GPW + grp; row0 < a.n;
         row0 += rows_per_iter * U) {
      long long idx[U];
      int k0[U], len[U];
      int maxlen = 0;
      XT acc[U], xi[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long row = row0 + u * rows_per_iter;
        idx[u] = row < a.n ? row * R + c : -1;
        acc[u] = zero<XT>();
        xi[u] = zero<XT>();
        k0[u] = 0;
        len[u] = 0;
        if (idx[u] >= 0) {
          k0[u] = __ldg(a.rowptr + row);
          len[u] = __ldg(a.rowptr + row + 1) - k0[u];
          xi[u] = in[idx[u]];
          if (K == MR_SPMM) xi[u] = sscal(sc, xi[u]);
        }
        maxlen = max(maxlen, len[u]);
      }
      for (int qq = 0; qq < maxlen; qq += 4) {
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (qq + tt < len[u]) {
              const int kk = k0[u] + qq + tt;
              const int col = __ldg(a.colidx + kk);
              const VT mv = __ldg(vals + kk);
              XT xv = in[(long long)col * R + c];
              if (K == MR_SPMM) xv = sscal(sc, xv);
              acc[u] = fma_(mv, xv, acc[u]);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (idx[u] < 0 || !on) continue;
        XT yv = acc[u];
        if (SIGMA) yv = fma_(from_c<XT>(a.sigma), xi[u], yv);
        if (K == MR_SPMM) {
          vout[idx[u]] = xi[u];
          if (sub_r1) yv = sub(yv, sscal(cb, r1[idx[u]]));
          out[idx[u]] = yv;
          q += to_c(cfma(xi[u], yv, zero<XT>())).x;   // Re <v, y>
        } else {
          const XT rv = sub(b[idx[u]], yv);
          if (K == MR_RESID) out[idx[u]] = rv;
          q += abs2(rv);
        }
      }
    }
  }
  __shared__ double tot_s[8];
  double qa[1] = {q};
  if (part_reduce<R, 1>(st.part, st.pstride, st.ticket, qa, grp, c, lane_ok, tot_s)) {
    mr_finish(st, K, tot_s);
    __syncthreads();
    if (threadIdx.x == 0) *st.ticket = 0u;
  }
}

}  // namespace sad
