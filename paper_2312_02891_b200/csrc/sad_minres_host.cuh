// sad_minres_host.cuh -- C-ABI of the device MINRES (sad_minres.cuh), included
// at the end of sad_capi.cu.  The reference's inner solver for Hermitian sides
// (krylov.py:271-287, minres(InnerSolveRequest(...)) behind SolverBinding.solve
// when uses_minres(shift), adi.py:468-488) on n x r blocks.
#pragma once

#include "sad_minres.cuh"

namespace sad {
int minres_launch_vec_d(int K, const MArgs& a, int R, int grid, cudaStream_t s);
int minres_launch_vec_z(int K, const MArgs& a, int R, int grid, cudaStream_t s);
int minres_launch_spmm_d(int K, const MArgs& a, int R, bool vc, bool sigma, int grid, cudaStream_t s);
int minres_launch_spmm_z(int K, const MArgs& a, int R, bool vc, bool sigma, int grid, cudaStream_t s);
}  // namespace sad

struct sad_minres {
  sad_ctx* ctx = nullptr;
  long long n = 0;
  int R = 1, dtype = 0;
  size_t esz = 8;
  char* vecs = nullptr;          // r1 r2 y t v w w2 (n x R each)
  char* state = nullptr;
  double* part = nullptr;
  int max_blocks = 0;
  long long* hflag_host = nullptr;
  long long* hflag_dev = nullptr;
  MState st{};
  int64_t bytes = 0;
};

extern "C" int sad_minres_destroy(sad_minres* w) {
  if (!w) return SAD_OK;
  ctx_free(w->ctx, w->vecs);
  ctx_free(w->ctx, w->state);
  ctx_free(w->ctx, w->part);
  if (w->hflag_host) cudaFreeHost(w->hflag_host);
  delete w;
  return SAD_OK;
}

extern "C" int sad_minres_create(sad_ctx* ctx, int64_t n, int r, int dtype, sad_minres** out) {
  if (!ctx || !out) return SAD_EINVAL;
  *out = nullptr;
  int rc = check_block(ctx, r, dtype);
  if (rc) return rc;
  if (n < 1) return set_err(ctx, SAD_EINVAL, "n must be >= 1");
  sad_minres* w = new sad_minres();
  w->ctx = ctx;
  w->n = n;
  w->R = r;
  w->dtype = dtype;
  w->esz = dtype == SAD_F64 ? 8 : 16;
  const size_t blk = ((size_t)n * r * w->esz + 255) & ~size_t(255);
  w->max_blocks = ctx->nsm * 8;
  const int pstride = 2 * 8;
  const size_t sb = (size_t)r * (14 * 8 + 8 + 5 * 4) + 16 * 8 + 256;
  if (ctx_malloc(ctx, (void**)&w->vecs, blk * 7) != cudaSuccess ||
      ctx_malloc(ctx, (void**)&w->state, sb) != cudaSuccess ||
      ctx_malloc(ctx, (void**)&w->part, (size_t)w->max_blocks * pstride * sizeof(double)) != cudaSuccess ||
      cudaHostAlloc(&w->hflag_host, 8 * sizeof(long long), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&w->hflag_dev, w->hflag_host, 0) != cudaSuccess) {
    sad_minres_destroy(w);
    return set_err(ctx, SAD_ENOMEM, "MINRES workspace allocation failed");
  }
  cudaMemset(w->state, 0, sb);
  char* p = w->state;
  MState& st = w->st;
  st.beta = carve<double>(p, r);
  st.oldb = carve<double>(p, r);
  st.dbar = carve<double>(p, r);
  st.epsln = carve<double>(p, r);
  st.phibar = carve<double>(p, r);
  st.cs = carve<double>(p, r);
  st.sn = carve<double>(p, r);
  st.check_at = carve<double>(p, r);
  st.alfa = carve<double>(p, r);
  st.c_oldeps = carve<double>(p, r);
  st.c_delta = carve<double>(p, r);
  st.c_gamma = carve<double>(p, r);
  st.c_phi = carve<double>(p, r);
  st.tnorm = carve<double>(p, r);
  st.it = carve<long long>(p, r);
  st.active = carve<int>(p, r);
  st.upd = carve<int>(p, r);
  st.chk = carve<int>(p, r);
  st.stop = carve<int>(p, r);
  st.any_chk = carve<int>(p, 1);
  st.err = carve<int>(p, 1);
  st.ticket = carve<unsigned>(p, 1);
  st.stepseq = carve<unsigned long long>(p, 1);
  if ((size_t)(p - w->state) > sb) {
    sad_minres_destroy(w);
    return set_err(ctx, SAD_EINVAL, "internal: MINRES state carve overflow");
  }
  st.part = w->part;
  st.hflag = reinterpret_cast<volatile long long*>(w->hflag_dev);
  st.R = r;
  st.pstride = pstride;
  w->bytes = (int64_t)(blk * 7 + sb + (size_t)w->max_blocks * pstride * 8);
  *out = w;
  return SAD_OK;
}

static __global__ void k_mr_init(MState st) {
  if (threadIdx.x < st.R) {
    st.it[threadIdx.x] = 0;
    st.active[threadIdx.x] = 0;
    st.upd[threadIdx.x] = 0;
    st.chk[threadIdx.x] = 0;
    st.stop[threadIdx.x] = 0;
    st.tnorm[threadIdx.x] = 0.0;
  }
  if (threadIdx.x == 0) {
    *st.any_chk = 0;
    *st.err = 0;
    *st.ticket = 0u;
    *st.stepseq = 0ull;
  }
}

extern "C" int sad_minres_solve_pc(sad_minres* w, sad_op* op, sad_pc* pc, const void* rhs, void* x,
                                   void* res, double tol_col, int maxit, void* stream,
                                   int64_t* iters_host, double* resnorm_host, uint8_t* conv_host);

extern "C" int sad_minres_solve(sad_minres* w, sad_op* op, const void* rhs, void* x, void* res,
                                double tol_col, int maxit, void* stream, int64_t* iters_host,
                                double* resnorm_host, uint8_t* conv_host) {
  return sad_minres_solve_pc(w, op, nullptr, rhs, x, res, tol_col, maxit, stream, iters_host,
                             resnorm_host, conv_host);
}

// pc != nullptr: the SPD split of an incomplete Cholesky factorisation,
// psolve = (G G^H)^-1 (apply_spd, precond.py:242-256; krylov.py:197-199)
extern "C" int sad_minres_solve_pc(sad_minres* w, sad_op* op, sad_pc* pc, const void* rhs, void* x,
                                   void* res, double tol_col, int maxit, void* stream,
                                   int64_t* iters_host, double* resnorm_host, uint8_t* conv_host) {
  if (!w) return SAD_EINVAL;
  sad_ctx* ctx = w->ctx;
  if (!op || !rhs || !x) return set_err(ctx, SAD_EINVAL, "null argument");
  if (!(tol_col > 0.0)) return set_err(ctx, SAD_EINVAL, "abs_tolerance must be positive");
  if (maxit < 0) return set_err(ctx, SAD_EINVAL, "maxit must be >= 0");
  if (op->n != w->n || op->ncols != w->n)
    return set_err(ctx, SAD_EINVAL, "operator size %lld != workspace size %lld", op->n, w->n);
  if (!op->real_ok || op->vals_complex)
    return set_err(ctx, SAD_EINVAL, "MINRES needs a real shift (Hermitian operator), adi.py:468-472");
  if (pc) {
    if (pc->n != w->n) return set_err(ctx, SAD_EINVAL, "preconditioner size != workspace size");
    if (pc->kind != SAD_PRECOND_IC0 && pc->kind != SAD_PRECOND_ICT)
      return set_err(ctx, SAD_EINVAL, "MINRES needs an SPD split (ic0 / ict), adi.py:468-472");
    if (pc->cplx) return set_err(ctx, SAD_EINVAL, "MINRES needs real Cholesky factors");
  }
  cudaStream_t s = S_(stream);
  const int R = w->R;
  const size_t blkb = (size_t)w->n * R * w->esz;
  const size_t blk = (blkb + 255) & ~size_t(255);
  MArgs a{};
  a.n = w->n;
  a.rowptr = op->rowptr;
  a.colidx = op->colidx;
  a.vals = op->vals;
  a.sigma = op->sigma_eff;
  a.dinv = w->dtype == SAD_F64 ? (const void*)op->dinv_r : (const void*)op->dinv_c;
  a.b = rhs;
  a.x = x;
  char* r1 = w->vecs;
  char* r2 = w->vecs + blk;
  a.y = w->vecs + 2 * blk;
  a.t = w->vecs + 3 * blk;
  a.v = w->vecs + 4 * blk;
  a.w = w->vecs + 5 * blk;
  a.w2 = w->vecs + 6 * blk;
  w->st.tol = tol_col;
  w->st.maxit = maxit;
  a.st = w->st;
  const int gpw = 32 / R;
  const int grid = grid_for(w->n, kWarps * gpw, std::min(w->max_blocks, ctx->nsm * 4));
  const bool cplx = w->dtype == SAD_C128;
  auto vec1 = [&](int K, int pmode) {
    a.r1 = r1;
    a.r2 = r2;
    a.pmode = pmode;
    return cplx ? minres_launch_vec_z(K, a, R, grid, s) : minres_launch_vec_d(K, a, R, grid, s);
  };
  // START / YUPD: with a Cholesky split, the vector part, y = (G G^H)^-1 y on the
  // device, then the dots and the finisher
  int pc_rc = SAD_OK;
  auto vec = [&](int K) {
    if (!pc || K == MR_WUPD) return vec1(K, 0);
    if (vec1(K, 1)) return 1;
    pc_rc = sad_pc_apply(pc, R, w->dtype, a.y, a.y, 1, s);
    if (pc_rc) return 1;
    return vec1(K, 2);
  };
  auto spmm = [&](int K) {
    a.r1 = r1;
    a.r2 = r2;
    return cplx ? minres_launch_spmm_z(K, a, R, op->vals_complex, op->sigma_identity, grid, s)
                : minres_launch_spmm_d(K, a, R, op->vals_complex, op->sigma_identity, grid, s);
  };
  volatile long long* hf = w->hflag_host;
  for (int i = 0; i < 8; ++i) hf[i] = -1;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  k_mr_init<<<1, 32, 0, s>>>(w->st);
  COUNT_LAUNCH(1);
  if (vec(MR_START)) return pc_rc ? pc_rc : set_err(ctx, SAD_EINVAL, "unsupported block width");
  const int LAG = 3;
  for (long long step = 0;; ++step) {
    bool stop = false;
    int rc = spin_until(ctx, s, [&] {
      const long long done = hf[0] < 0 ? 0 : hf[0];
      if (done >= 1 && hf[1] == 0) { stop = true; return true; }
      return step - done <= LAG;
    });
    if (rc) return rc;
    if (stop || step >= (long long)maxit + LAG + 1) break;
    // the first iterations are issued before any flag can say "stop": a column
    // that has ended leaves them as no-ops (gated on its flags)
    if (spmm(MR_SPMM) || vec(MR_YUPD))
      return pc_rc ? pc_rc : set_err(ctx, SAD_EINVAL, "unsupported block width / value type");
    std::swap(r1, r2);     // r1 <- old r2, r2 <- the new residual (written into old r1)
    if (vec(MR_WUPD) || spmm(MR_CHECK))
      return set_err(ctx, SAD_EINVAL, "unsupported block width / value type");
    CKL(ctx);
  }
  spmm(MR_RESID);
  CKL(ctx);
  if (res) CK(ctx, cudaMemcpyAsync(res, a.t, blkb, cudaMemcpyDeviceToDevice, s));
  std::vector<long long> it(R);
  std::vector<double> tn(R);
  int err = 0;
  CK(ctx, cudaMemcpyAsync(it.data(), w->st.it, R * sizeof(long long), cudaMemcpyDeviceToHost, s));
  CK(ctx, cudaMemcpyAsync(tn.data(), w->st.tnorm, R * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(ctx, cudaMemcpyAsync(&err, w->st.err, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(ctx, cudaStreamSynchronize(s));
  if (err)
    return set_err(ctx, SAD_EBREAKDOWN,
                   "MINRES preconditioner is not positive definite (<b, P b> = %g)", tn[0]);
  for (int c = 0; c < R; ++c) {
    if (iters_host) iters_host[c] = it[c];
    if (resnorm_host) resnorm_host[c] = tn[c];
    if (conv_host) conv_host[c] = tn[c] <= tol_col ? 1 : 0;
  }
  return SAD_OK;
}

extern "C" int64_t sad_minres_bytes(const sad_minres* w) { return w ? w->bytes : -1; }
