// sad_precond_host.cuh -- C-ABI of the incomplete-factorisation preconditioners,
// included at the end of sad_capi.cu.
//
// sad_pc_create builds, ONCE per distinct shift (the reference's factorisation
// cache, adi.py:453-466), what precond.py:307-357 `factorize` builds: the
// assembled shifted matrix (sparse.py:138-155, conjugate-transposed on the B
// side), the row-wise IKJ incomplete LU with threshold dropping or pattern
// restriction (precond.py:34-125) and, for the Cholesky kinds, the fold
// G = L sqrt(D) (precond.py:279-304).  The factorisation is a sequential
// recurrence with a data-dependent pattern, so it runs on the host (a sparse
// accumulator with a heap of pending pivots instead of the reference's dense
// scans, same arithmetic in the same order: the factors are bit-identical to
// the reference's).  What the Krylov iteration calls thousands of times -- the
// triangular solves -- runs on the device (sad_precond.cuh): the factors are
// uploaded in solve order together with their level schedules.
#pragma once

#include <queue>

#include "sad_precond.cuh"

namespace sad {
int sptrsv_launch(const TriArgs& a, int R, bool block_complex, bool vals_complex, int grid,
                  cudaStream_t s);
}

namespace {

struct HC { double re, im; };   // host complex, arithmetic spelled out (no fma, numba's order)
inline HC hc_mul(HC a, HC b) {
  const double ac = a.re * b.re, bd = a.im * b.im, ad = a.re * b.im, bc = a.im * b.re;
  return HC{ac - bd, ad + bc};
}
inline HC hc_sub(HC a, HC b) { return HC{a.re - b.re, a.im - b.im}; }
inline HC hc_div(HC a, HC b) {   // CPython's _Py_c_quot (numba's complex128 quotient)
  if (std::fabs(b.re) >= std::fabs(b.im)) {
    if (b.re == 0.0) return HC{NAN, NAN};
    const double ratio = b.im / b.re, denom = b.re + b.im * ratio;
    return HC{(a.re + a.im * ratio) / denom, (a.im - a.re * ratio) / denom};
  }
  const double ratio = b.re / b.im, denom = b.re * ratio + b.im;
  return HC{(a.re * ratio + a.im) / denom, (a.im * ratio - a.re) / denom};
}
inline double hc_abs(HC a) { return std::hypot(a.re, a.im); }

struct HostCsrZ {   // complex CSR on the host (the reference's int64/complex128 triplets)
  std::vector<int64_t> ptr, idx;
  std::vector<HC> val;
};

// base + sigma*mass on the merged pattern, entries that cancel exactly dropped
// (scipy's csr_plus_csr keeps nonzero sums only); mass == nullptr: identity
void assemble_host(long long n, const std::vector<int>& brp, const std::vector<int>& bci,
                   const std::vector<double>& bv, const std::vector<int>* mrp,
                   const std::vector<int>* mci, const std::vector<double>* mv, double2 sig,
                   HostCsrZ& out) {
  out.ptr.assign(n + 1, 0);
  out.idx.clear();
  out.val.clear();
  out.idx.reserve(bci.size() + (size_t)n);
  out.val.reserve(bci.size() + (size_t)n);
  const bool cplx = sig.y != 0.0;
  for (long long i = 0; i < n; ++i) {
    int p = brp[i];
    const int pe = brp[i + 1];
    int q = mrp ? (*mrp)[i] : 0;
    const int qe = mrp ? (*mrp)[i + 1] : 1;
    while (p < pe || q < qe) {
      const long long cb = p < pe ? bci[p] : (long long)INT32_MAX;
      const long long cm = q < qe ? (mrp ? (long long)(*mci)[q] : i) : (long long)INT32_MAX;
      const long long col = std::min(cb, cm);
      double a = 0.0, mm = 0.0;
      bool hb = false, hm = false;
      if (cb == col) { a = bv[p++]; hb = true; }
      if (cm == col) { mm = mrp ? (*mv)[q] : 1.0; ++q; hm = true; }
      HC v;
      if (!cplx) {
        // real shift: base + shift.real * mass in real arithmetic
        v.re = hm ? (hb ? a + sig.x * mm : sig.x * mm) : a;
        v.im = 0.0;
      } else {
        // complex shift: base.astype(complex) + shift * mass
        const HC sm = hm ? HC{sig.x * mm, sig.y * mm} : HC{0.0, 0.0};
        v.re = hb ? (hm ? a + sm.re : a) : sm.re;
        v.im = hb ? (hm ? 0.0 + sm.im : 0.0) : sm.im;
      }
      if (v.re == 0.0 && v.im == 0.0) continue;
      out.idx.push_back(col);
      out.val.push_back(v);
    }
    out.ptr[i + 1] = (int64_t)out.idx.size();
  }
}

struct IluOut {
  HostCsrZ L, U;   // L unit lower without diagonal; U upper, diagonal first in each row
  int status = 0;
};

// precond.py:34-125 with a sparse accumulator: the pending pivots k < i of row i
// live in a min-heap (fill only appears right of the pivot being eliminated, so
// popping the heap visits them in the reference's increasing-k order).
void ilu_host(long long n, const HostCsrZ& A, double droptol, bool restrict_pattern, IluOut& out) {
  std::vector<HC> w(n, HC{0.0, 0.0});
  std::vector<char> occ(n, 0), inpat(n, 0);
  std::vector<HC> udiag(n, HC{0.0, 0.0});
  std::vector<int64_t> touched, keep;
  std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> heap;
  out.L.ptr.assign(n + 1, 0);
  out.U.ptr.assign(n + 1, 0);
  out.status = 0;
  for (long long i = 0; i < n; ++i) {
    double rownorm = 0.0;
    touched.clear();
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p) {
      const int64_t j = A.idx[p];
      const HC v = A.val[p];
      w[j] = v;
      if (!occ[j]) {
        occ[j] = 1;
        touched.push_back(j);
        if (j < i) heap.push(j);
      }
      inpat[j] = 1;
      rownorm += (v.re * v.re + v.im * v.im);
    }
    const double tau = droptol * std::sqrt(rownorm);
    while (!heap.empty()) {
      const int64_t k = heap.top();
      heap.pop();
      const HC lik = hc_div(w[k], udiag[k]);
      if (!restrict_pattern && hc_abs(lik) < tau) {
        w[k] = HC{0.0, 0.0};
        occ[k] = 0;
        continue;
      }
      w[k] = lik;
      for (int64_t p = out.U.ptr[k] + 1; p < out.U.ptr[k + 1]; ++p) {
        const int64_t j = out.U.idx[p];
        if (restrict_pattern && !inpat[j]) continue;
        w[j] = hc_sub(w[j], hc_mul(lik, out.U.val[p]));
        if (!occ[j]) {
          occ[j] = 1;
          touched.push_back(j);
          if (j < i) heap.push(j);
        }
      }
    }
    const HC piv = w[i];
    if (hc_abs(piv) < 1e-300) {   // precond.py:17, 89-92
      out.status = 1;
      return;
    }
    udiag[i] = piv;
    std::sort(touched.begin(), touched.end());
    for (int64_t j : touched)
      if (j < i && occ[j]) {
        out.L.idx.push_back(j);
        out.L.val.push_back(w[j]);
      }
    out.L.ptr[i + 1] = (int64_t)out.L.idx.size();
    out.U.idx.push_back(i);
    out.U.val.push_back(piv);
    for (int64_t j : touched)
      if (j > i && occ[j] && (restrict_pattern || hc_abs(w[j]) >= tau)) {
        out.U.idx.push_back(j);
        out.U.val.push_back(w[j]);
      }
    out.U.ptr[i + 1] = (int64_t)out.U.idx.size();
    for (int64_t j : touched) {
      w[j] = HC{0.0, 0.0};
      occ[j] = 0;
      inpat[j] = 0;
    }
  }
}

// One triangular factor on the device, in solve order
struct TriFactor {
  long long n = 0, nnz = 0;
  int* rowptr = nullptr;
  int* colidx = nullptr;
  void* vals = nullptr;
  void* diag = nullptr;        // nullptr: unit diagonal
  bool vals_complex = false;
  int levels = 0;
  std::vector<int> level_rows;  // rows sorted by level (host)
  std::vector<int> level_ptr;   // [levels + 1]
  // schedules per lane-group count 32/R (built on demand)
  struct Sched { int* order = nullptr; int ntasks = 0; };
  std::map<int, Sched> sched;
  void* cells = nullptr;       // 16-byte {value, epoch} cells of the solved elements
  size_t cells_cap = 0;        // cells allocated
  long long epoch = 0;
  unsigned* counter = nullptr;
};

}  // namespace

struct sad_pc {
  sad_ctx* ctx = nullptr;
  long long n = 0;
  int kind = 0;
  double droptol = 0.0;
  double sign = 1.0;
  bool cplx = false;            // factor values complex
  // the reference's layout, kept on the host for sad_pc_get_factor
  HostCsrZ L, U, G;
  TriFactor f1, f2;             // ILU: L then U; Cholesky: G then G^T
};

namespace {

void tri_free(sad_ctx* ctx, TriFactor& f) {
  ctx_free(ctx, f.rowptr);
  ctx_free(ctx, f.colidx);
  ctx_free(ctx, f.vals);
  ctx_free(ctx, f.diag);
  ctx_free(ctx, f.cells);
  ctx_free(ctx, f.counter);
  for (auto& kv : f.sched) ctx_free(ctx, kv.second.order);
  f = TriFactor();
}

// rows: off-diagonal entries (ptr/idx/val) in accumulation order; diag: per-row
// divisor or empty; lower: dependencies have smaller row indices
int tri_upload(sad_ctx* ctx, TriFactor& f, long long n, const std::vector<int64_t>& ptr,
               const std::vector<int64_t>& idx, const std::vector<HC>& val,
               const std::vector<HC>& diag, bool lower, bool cplx) {
  f.n = n;
  f.nnz = (long long)idx.size();
  f.vals_complex = cplx;
  std::vector<int> rp(n + 1), ci(idx.size());
  for (long long i = 0; i <= n; ++i) rp[i] = (int)ptr[i];
  for (size_t k = 0; k < idx.size(); ++k) ci[k] = (int)idx[k];
  // dependency levels
  std::vector<int> lev(n, 0);
  int nlev = 0;
  auto visit = [&](long long i) {
    int l = 0;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) l = std::max(l, lev[idx[p]] + 1);
    lev[i] = l;
    nlev = std::max(nlev, l + 1);
  };
  if (lower) for (long long i = 0; i < n; ++i) visit(i);
  else for (long long i = n - 1; i >= 0; --i) visit(i);
  f.levels = nlev;
  f.level_ptr.assign(nlev + 1, 0);
  for (long long i = 0; i < n; ++i) f.level_ptr[lev[i] + 1]++;
  for (int l = 0; l < nlev; ++l) f.level_ptr[l + 1] += f.level_ptr[l];
  f.level_rows.resize(n);
  {
    std::vector<int> pos(f.level_ptr.begin(), f.level_ptr.end() - 1);
    for (long long i = 0; i < n; ++i) f.level_rows[pos[lev[i]]++] = (int)i;
  }
  const size_t nz = std::max<size_t>(idx.size(), 1);
  const size_t esz = cplx ? sizeof(double2) : sizeof(double);
  CK(ctx, ctx_malloc(ctx, (void**)&f.rowptr, (n + 1) * sizeof(int)));
  CK(ctx, ctx_malloc(ctx, (void**)&f.colidx, nz * sizeof(int)));
  CK(ctx, ctx_malloc(ctx, &f.vals, nz * esz));
  CK(ctx, ctx_malloc(ctx, (void**)&f.counter, 256));
  CK(ctx, cudaMemcpy(f.rowptr, rp.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice));
  if (!idx.empty()) CK(ctx, cudaMemcpy(f.colidx, ci.data(), ci.size() * sizeof(int), cudaMemcpyHostToDevice));
  auto put = [&](void* dst, const std::vector<HC>& src) -> cudaError_t {
    if (src.empty()) return cudaSuccess;
    if (cplx) return cudaMemcpy(dst, src.data(), src.size() * sizeof(HC), cudaMemcpyHostToDevice);
    std::vector<double> re(src.size());
    for (size_t k = 0; k < src.size(); ++k) re[k] = src[k].re;
    return cudaMemcpy(dst, re.data(), re.size() * sizeof(double), cudaMemcpyHostToDevice);
  };
  CK(ctx, put(f.vals, val));
  if (!diag.empty()) {
    CK(ctx, ctx_malloc(ctx, &f.diag, (size_t)n * esz));
    CK(ctx, put(f.diag, diag));
  }
  return SAD_OK;
}

int tri_sched(sad_ctx* ctx, TriFactor& f, int gpw, TriFactor::Sched** out) {
  auto it = f.sched.find(gpw);
  if (it == f.sched.end()) {
    std::vector<int> order;
    order.reserve((size_t)f.n + (size_t)f.levels * gpw);
    for (int l = 0; l < f.levels; ++l) {
      for (int k = f.level_ptr[l]; k < f.level_ptr[l + 1]; ++k) order.push_back(f.level_rows[k]);
      while (order.size() % gpw) order.push_back(-1);
    }
    TriFactor::Sched s;
    s.ntasks = (int)(order.size() / gpw);
    CK(ctx, ctx_malloc(ctx, (void**)&s.order, std::max<size_t>(order.size(), 1) * sizeof(int)));
    if (!order.empty())
      CK(ctx, cudaMemcpy(s.order, order.data(), order.size() * sizeof(int), cudaMemcpyHostToDevice));
    it = f.sched.emplace(gpw, s).first;
  }
  *out = &it->second;
  return SAD_OK;
}

// x = T^{-1} (negate ? -b : b) on n x r blocks; x may alias b
int tri_solve(sad_ctx* ctx, TriFactor& f, int r, int dtype, const void* b, void* x, bool negate,
              cudaStream_t s) {
  TriFactor::Sched* sc = nullptr;
  int rc = tri_sched(ctx, f, 32 / r, &sc);
  if (rc) return rc;
  const size_t need = (size_t)f.n * r * (dtype == SAD_C128 ? 2 : 1);
  if (f.cells_cap < need) {
    // tags start below any epoch; a wider (or complex) block needs more cells
    CK(ctx, cudaStreamSynchronize(s));
    ctx_free(ctx, f.cells);
    f.cells = nullptr;
    CK(ctx, ctx_malloc(ctx, &f.cells, need * 16));
    CK(ctx, cudaMemsetAsync(f.cells, 0, need * 16, s));
    f.cells_cap = need;
    f.epoch = 0;
  }
  TriArgs a{};
  a.n = f.n;
  a.rowptr = f.rowptr;
  a.colidx = f.colidx;
  a.vals = f.vals;
  a.diag = f.diag;
  a.order = sc->order;
  a.ntasks = sc->ntasks;
  a.cells = f.cells;
  a.epoch = ++f.epoch;
  a.counter = f.counter;
  a.b = b;
  a.x = x;
  a.negate = negate ? 1 : 0;
  CK(ctx, cudaMemsetAsync(f.counter, 0, sizeof(unsigned), s));
  const int grid = std::max(1, std::min((sc->ntasks + kWarps - 1) / kWarps, ctx->nsm * 8));
  if (sptrsv_launch(a, r, dtype == SAD_C128, f.vals_complex, grid, s))
    return set_err(ctx, SAD_EINVAL, "complex factors need a complex128 block");
  CKL(ctx);
  return SAD_OK;
}

}  // namespace

extern "C" int sad_pc_destroy(sad_pc* pc) {
  if (!pc) return SAD_OK;
  tri_free(pc->ctx, pc->f1);
  tri_free(pc->ctx, pc->f2);
  delete pc;
  return SAD_OK;
}

extern "C" int sad_pc_create(sad_ctx* ctx, const sad_csr* base, const sad_csr* mass, double sre,
                             double sim, int adjoint, int kind, double droptol, sad_pc** out) {
  if (!ctx || !base || !out) return SAD_EINVAL;
  *out = nullptr;
  if (kind != SAD_PRECOND_ILU0 && kind != SAD_PRECOND_ILUT && kind != SAD_PRECOND_IC0 &&
      kind != SAD_PRECOND_ICT)
    return set_err(ctx, SAD_EINVAL, "sad_pc_create: kind %d is not an incomplete factorisation", kind);
  if (base->nrows != base->ncols) return set_err(ctx, SAD_EINVAL, "preconditioned matrix must be square");
  if (mass && (mass->nrows != base->nrows || mass->ncols != base->ncols))
    return set_err(ctx, SAD_EINVAL, "base and mass dimensions disagree");
  if (adjoint && (!base->has_t || (mass && !mass->has_t)))
    return set_err(ctx, SAD_EINVAL, "adjoint operator needs matrices created with build_transpose");
  const long long n = base->nrows;
  const double2 sig = adjoint ? make_double2(sre, -sim) : make_double2(sre, sim);
  HostCsrZ A;
  assemble_host(n, adjoint ? base->ht_rowptr : base->h_rowptr,
                adjoint ? base->ht_colidx : base->h_colidx, adjoint ? base->ht_vals : base->h_vals,
                mass ? (adjoint ? &mass->ht_rowptr : &mass->h_rowptr) : nullptr,
                mass ? (adjoint ? &mass->ht_colidx : &mass->h_colidx) : nullptr,
                mass ? (adjoint ? &mass->ht_vals : &mass->h_vals) : nullptr, sig, A);
  const bool chol = (kind == SAD_PRECOND_IC0 || kind == SAD_PRECOND_ICT);
  double sign = 1.0;
  if (chol) {
    // precond.py:340-346: a negative definite shifted matrix is negated first
    double dsum = 0.0;
    for (long long i = 0; i < n; ++i)
      for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p)
        if (A.idx[p] == i) dsum += A.val[p].re;
    if (dsum < 0.0) {
      sign = -1.0;
      for (HC& v : A.val) { v.re = -v.re; v.im = -v.im; }
    }
  }
  const bool restrict_pattern = (kind == SAD_PRECOND_ILU0 || kind == SAD_PRECOND_IC0);
  IluOut lu;
  ilu_host(n, A, restrict_pattern ? 0.0 : droptol, restrict_pattern, lu);
  if (lu.status != 0)
    return set_err(ctx, SAD_EBREAKDOWN, "zero pivot in %s factorization",
                   kind == SAD_PRECOND_ILU0 ? "ilu0" : kind == SAD_PRECOND_ILUT ? "ilut"
                   : kind == SAD_PRECOND_IC0 ? "ic0" : "ict");
  sad_pc* pc = new sad_pc();
  pc->ctx = ctx;
  pc->n = n;
  pc->kind = kind;
  pc->droptol = droptol;
  pc->sign = sign;
  int rc = SAD_OK;
  auto any_imag = [](const std::vector<HC>& v) {
    for (const HC& z : v)
      if (z.im != 0.0) return true;
    return false;
  };
  if (!chol) {
    pc->cplx = any_imag(lu.L.val) || any_imag(lu.U.val);
    // U in solve order: the diagonal (first entry) apart
    std::vector<int64_t> up(n + 1, 0), ui;
    std::vector<HC> uv, ud(n);
    ui.reserve(lu.U.idx.size());
    uv.reserve(lu.U.idx.size());
    for (long long i = 0; i < n; ++i) {
      ud[i] = lu.U.val[lu.U.ptr[i]];
      for (int64_t p = lu.U.ptr[i] + 1; p < lu.U.ptr[i + 1]; ++p) {
        ui.push_back(lu.U.idx[p]);
        uv.push_back(lu.U.val[p]);
      }
      up[i + 1] = (int64_t)ui.size();
    }
    rc = tri_upload(ctx, pc->f1, n, lu.L.ptr, lu.L.idx, lu.L.val, {}, true, pc->cplx);
    if (rc == SAD_OK) rc = tri_upload(ctx, pc->f2, n, up, ui, uv, ud, false, pc->cplx);
    pc->L = std::move(lu.L);
    pc->U = std::move(lu.U);
  } else {
    // precond.py:279-304: D = diag(U) must be real positive; G = L sqrt(D), diagonal last
    std::vector<double> sq(n);
    for (long long i = 0; i < n; ++i) {
      const HC d = lu.U.val[lu.U.ptr[i]];
      if (d.re <= 0.0 || std::fabs(d.im) > 1e-10 * std::fabs(d.re)) {
        delete pc;
        return set_err(ctx, SAD_EBREAKDOWN, "matrix is not positive definite up to dropping");
      }
      sq[i] = std::sqrt(d.re);
    }
    HostCsrZ& G = pc->G;
    G.ptr.assign(n + 1, 0);
    std::vector<int64_t> gp(n + 1, 0), gi;     // strictly lower part, solve order
    std::vector<HC> gv, gd(n);
    std::vector<int64_t> tcount(n + 1, 0);
    for (long long i = 0; i < n; ++i) {
      for (int64_t p = lu.L.ptr[i]; p < lu.L.ptr[i + 1]; ++p) {
        const int64_t j = lu.L.idx[p];
        const HC v = hc_mul(lu.L.val[p], HC{sq[j], 0.0});
        G.idx.push_back(j);
        G.val.push_back(v);
        gi.push_back(j);
        gv.push_back(v);
        tcount[j + 1]++;
      }
      G.idx.push_back(i);
      G.val.push_back(HC{sq[i], 0.0});
      G.ptr[i + 1] = (int64_t)G.idx.size();
      gp[i + 1] = (int64_t)gi.size();
      gd[i] = HC{sq[i], 0.0};
    }
    pc->cplx = any_imag(G.val);
    // G^T rows with descending column order: the order precond.py:165-173's scatter
    // solve (rows i = n-1 .. 0) updates entry b[j]
    std::vector<int64_t> tp(n + 1, 0), ti(gi.size());
    std::vector<HC> tv(gi.size());
    for (long long j = 0; j < n; ++j) tp[j + 1] = tp[j] + tcount[j + 1];
    {
      std::vector<int64_t> pos(tp.begin(), tp.end() - 1);
      for (long long i = n - 1; i >= 0; --i)
        for (int64_t p = gp[i]; p < gp[i + 1]; ++p) {
          const int64_t j = gi[p];
          ti[pos[j]] = i;
          tv[pos[j]] = gv[p];
          pos[j]++;
        }
    }
    rc = tri_upload(ctx, pc->f1, n, gp, gi, gv, gd, true, pc->cplx);
    if (rc == SAD_OK) rc = tri_upload(ctx, pc->f2, n, tp, ti, tv, gd, false, pc->cplx);
  }
  if (rc != SAD_OK) {
    sad_pc_destroy(pc);
    return rc;
  }
  *out = pc;
  return SAD_OK;
}

// info[8]: kind, n, nnz of the first / second factor (reference layout), complex
// factors, dependency levels of the first / second solve, sign
extern "C" int sad_pc_info(const sad_pc* pc, int64_t* info) {
  if (!pc || !info) return SAD_EINVAL;
  const bool chol = (pc->kind == SAD_PRECOND_IC0 || pc->kind == SAD_PRECOND_ICT);
  info[0] = pc->kind;
  info[1] = pc->n;
  info[2] = chol ? (int64_t)pc->G.idx.size() : (int64_t)pc->L.idx.size();
  info[3] = chol ? 0 : (int64_t)pc->U.idx.size();
  info[4] = pc->cplx ? 1 : 0;
  info[5] = pc->f1.levels;
  info[6] = pc->f2.levels;
  info[7] = pc->sign < 0 ? -1 : 1;
  return SAD_OK;
}

// which: 0 = L (unit lower, no diagonal) / G (lower, diagonal last); 1 = U (upper,
// diagonal first) -- the reference's raw triplets (precond.py:124-125, 288-302)
extern "C" int sad_pc_get_factor(const sad_pc* pc, int which, int64_t* indptr, int64_t* indices,
                                 double* data_ri) {
  if (!pc || !indptr || !indices || !data_ri) return SAD_EINVAL;
  const bool chol = (pc->kind == SAD_PRECOND_IC0 || pc->kind == SAD_PRECOND_ICT);
  const HostCsrZ* f = chol ? (which == 0 ? &pc->G : nullptr) : (which == 0 ? &pc->L : &pc->U);
  if (!f) return set_err(pc->ctx, SAD_EINVAL, "Cholesky kinds store one factor");
  std::memcpy(indptr, f->ptr.data(), f->ptr.size() * sizeof(int64_t));
  if (!f->idx.empty()) {
    std::memcpy(indices, f->idx.data(), f->idx.size() * sizeof(int64_t));
    std::memcpy(data_ri, f->val.data(), f->val.size() * sizeof(HC));
  }
  return SAD_OK;
}

// y = M^{-1} x: IncompleteFactorization.apply (precond.py:224-240), or with
// spd != 0 apply_spd (precond.py:242-256, Cholesky kinds only).  y may alias x.
extern "C" int sad_pc_apply(sad_pc* pc, int r, int dtype, const void* x, void* y, int spd,
                            void* stream) {
  if (!pc) return SAD_EINVAL;
  sad_ctx* ctx = pc->ctx;
  if (!x || !y) return set_err(ctx, SAD_EINVAL, "null argument");
  int rc = check_block(ctx, r, dtype);
  if (rc) return rc;
  const bool chol = (pc->kind == SAD_PRECOND_IC0 || pc->kind == SAD_PRECOND_ICT);
  if (spd && !chol) return set_err(ctx, SAD_EINVAL, "this kind has no SPD split form");
  if (pc->cplx && dtype != SAD_C128)
    return set_err(ctx, SAD_EINVAL, "complex factors need a complex128 block");
  cudaStream_t s = S_(stream);
  const bool neg = chol && !spd && pc->sign < 0;   // -(G G^T)^{-1} x = (G G^T)^{-1} (-x), exactly
  rc = tri_solve(ctx, pc->f1, r, dtype, x, y, neg, s);
  if (rc) return rc;
  return tri_solve(ctx, pc->f2, r, dtype, y, y, false, s);
}
