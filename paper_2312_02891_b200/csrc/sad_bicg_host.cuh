// sad_bicg_host.cuh -- C-ABI of the device BiCGstab (sad_bicg.cuh), included
// at the end of sad_capi.cu.  The reference's default inner solver
// (krylov.py:160-184, bicgstab(InnerSolveRequest(...)) behind
// SolverBinding.solve, adi.py:473-488) on n x r blocks.
#pragma once

#include "sad_bicg.cuh"

namespace sad {
int bicg_launch_vec_d(int K, const BArgs& a, int R, int grid, cudaStream_t s);
int bicg_launch_vec_z(int K, const BArgs& a, int R, int grid, cudaStream_t s);
int bicg_launch_spmm_d(int K, const BArgs& a, int R, bool vc, bool sigma, int grid, cudaStream_t s);
int bicg_launch_spmm_z(int K, const BArgs& a, int R, bool vc, bool sigma, int grid, cudaStream_t s);
}  // namespace sad

struct sad_bicg {
  sad_ctx* ctx = nullptr;
  long long n = 0;
  int R = 1, dtype = 0;
  size_t esz = 8;
  char* vecs = nullptr;          // dx r rhat p v s t (n x R each)
  char* pvecs = nullptr;         // phat shat (general preconditioners; lazy)
  char* state = nullptr;
  double* part = nullptr;
  int max_blocks = 0;
  long long* hflag_host = nullptr;
  long long* hflag_dev = nullptr;
  BState st{};
  int64_t bytes = 0;
};

extern "C" int sad_bicg_create(sad_ctx* ctx, int64_t n, int r, int dtype, sad_bicg** out) {
  if (!ctx || !out) return SAD_EINVAL;
  *out = nullptr;
  int rc = check_block(ctx, r, dtype);
  if (rc) return rc;
  if (n < 1) return set_err(ctx, SAD_EINVAL, "n must be >= 1");
  sad_bicg* w = new sad_bicg();
  w->ctx = ctx;
  w->n = n;
  w->R = r;
  w->dtype = dtype;
  w->esz = dtype == SAD_F64 ? 8 : 16;
  const size_t blk = ((size_t)n * r * w->esz + 255) & ~size_t(255);
  w->max_blocks = ctx->nsm * 8;
  const int pstride = 5 * 8;
  size_t sb = (size_t)r * (5 * 16 + 3 * 8 + 2 * 8 + 8 * 4) + 16 * 8 + 256;
  if (ctx_malloc(ctx, (void**)&w->vecs, blk * 7) != cudaSuccess ||
      ctx_malloc(ctx, (void**)&w->state, sb) != cudaSuccess ||
      ctx_malloc(ctx, (void**)&w->part, (size_t)w->max_blocks * pstride * sizeof(double)) != cudaSuccess ||
      cudaHostAlloc(&w->hflag_host, 8 * sizeof(long long), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&w->hflag_dev, w->hflag_host, 0) != cudaSuccess) {
    ctx_free(ctx, w->vecs);
    ctx_free(ctx, w->state);
    ctx_free(ctx, w->part);
    if (w->hflag_host) cudaFreeHost(w->hflag_host);
    delete w;
    return set_err(ctx, SAD_ENOMEM, "BiCGstab workspace allocation failed");
  }
  cudaMemset(w->state, 0, sb);
  char* p = w->state;
  BState& st = w->st;
  st.rho = carve<double2>(p, r);
  st.alpha = carve<double2>(p, r);
  st.omega = carve<double2>(p, r);
  st.rho_new = carve<double2>(p, r);
  st.beta = carve<double2>(p, r);
  st.scale = carve<double>(p, r);
  st.nr2 = carve<double>(p, r);
  st.tnorm = carve<double>(p, r);
  st.it = carve<long long>(p, r);
  st.run_it = carve<long long>(p, r);
  st.active = carve<int>(p, r);
  st.ok = carve<int>(p, r);
  st.skip = carve<int>(p, r);
  st.fresh = carve<int>(p, r);
  st.rmode = carve<int>(p, r);
  st.restarted = carve<int>(p, r);
  st.inrun = carve<int>(p, r);
  st.any_active = carve<int>(p, 1);
  st.ticket = carve<unsigned>(p, 1);
  st.stepseq = carve<unsigned long long>(p, 1);
  st.cycleseq = carve<unsigned long long>(p, 1);
  if ((size_t)(p - w->state) > sb) {
    sad_bicg_destroy(w);
    return set_err(ctx, SAD_EINVAL, "internal: BiCGstab state carve overflow");
  }
  st.part = w->part;
  st.hflag = reinterpret_cast<volatile long long*>(w->hflag_dev);
  st.R = r;
  st.pstride = pstride;
  w->bytes = (int64_t)(blk * 7 + sb + (size_t)w->max_blocks * pstride * 8);
  *out = w;
  return SAD_OK;
}

extern "C" int sad_bicg_destroy(sad_bicg* w) {
  if (!w) return SAD_OK;
  ctx_free(w->ctx, w->vecs);
  ctx_free(w->ctx, w->pvecs);
  ctx_free(w->ctx, w->state);
  ctx_free(w->ctx, w->part);
  if (w->hflag_host) cudaFreeHost(w->hflag_host);
  delete w;
  return SAD_OK;
}

// solve start: flags, counters; every column takes part in the first run
static __global__ void k_bi_init(BState st) {
  if (threadIdx.x < st.R) {
    const int c = threadIdx.x;
    st.it[c] = 0;
    st.run_it[c] = 0;
    st.active[c] = 0;
    st.ok[c] = 0;
    st.skip[c] = 0;
    st.fresh[c] = 0;
    st.rmode[c] = 0;
    st.restarted[c] = 0;
    st.inrun[c] = 1;
    st.tnorm[c] = 0.0;
  }
  if (threadIdx.x == 0) {
    *st.any_active = 0;
    *st.ticket = 0u;
    *st.stepseq = 0ull;
    *st.cycleseq = 0ull;
  }
}

extern "C" int sad_bicg_solve_pc(sad_bicg* w, sad_op* op, sad_pc* pc, const void* rhs, void* x,
                                 void* res, double tol_col, int maxit, void* stream,
                                 int64_t* iters_host, double* resnorm_host, uint8_t* conv_host);

extern "C" int sad_bicg_solve(sad_bicg* w, sad_op* op, const void* rhs, void* x, void* res,
                              double tol_col, int maxit, void* stream, int64_t* iters_host,
                              double* resnorm_host, uint8_t* conv_host) {
  return sad_bicg_solve_pc(w, op, nullptr, rhs, x, res, tol_col, maxit, stream, iters_host,
                           resnorm_host, conv_host);
}

// pc != nullptr: right preconditioning by an incomplete factorisation
// (_precond_apply, krylov.py:73-76); the operator must carry no Jacobi scaling
extern "C" int sad_bicg_solve_pc(sad_bicg* w, sad_op* op, sad_pc* pc, const void* rhs, void* x,
                                 void* res, double tol_col, int maxit, void* stream,
                                 int64_t* iters_host, double* resnorm_host, uint8_t* conv_host) {
  if (!w) return SAD_EINVAL;
  sad_ctx* ctx = w->ctx;
  if (!op || !rhs || !x) return set_err(ctx, SAD_EINVAL, "null argument");
  if (!(tol_col > 0.0)) return set_err(ctx, SAD_EINVAL, "abs_tolerance must be positive");
  if (maxit < 0) return set_err(ctx, SAD_EINVAL, "maxit must be >= 0");
  if (op->n != w->n || op->ncols != w->n)
    return set_err(ctx, SAD_EINVAL, "operator size %lld != workspace size %lld", op->n, w->n);
  if (w->dtype == SAD_F64 && !op->real_ok)
    return set_err(ctx, SAD_EINVAL, "complex shift needs a complex128 workspace");
  cudaStream_t s = S_(stream);
  const int R = w->R;
  const size_t blkb = (size_t)w->n * R * w->esz;
  const size_t blk = (blkb + 255) & ~size_t(255);
  BArgs a{};
  a.n = w->n;
  a.rowptr = op->rowptr;
  a.colidx = op->colidx;
  a.vals = op->vals;
  a.sigma = op->sigma_eff;
  a.dinv = w->dtype == SAD_F64 ? (const void*)op->dinv_r : (const void*)op->dinv_c;
  a.b = rhs;
  a.x = x;
  a.dx = w->vecs;
  a.r = w->vecs + blk;
  a.rhat = w->vecs + 2 * blk;
  a.p = w->vecs + 3 * blk;
  a.v = w->vecs + 4 * blk;
  a.s = w->vecs + 5 * blk;
  a.t = w->vecs + 6 * blk;
  if (pc) {
    if (pc->n != w->n) return set_err(ctx, SAD_EINVAL, "preconditioner size != workspace size");
    if (op->precond != SAD_PRECOND_NONE)
      return set_err(ctx, SAD_EINVAL, "an operator used with sad_pc must be created with SAD_PRECOND_NONE");
    if (pc->cplx && w->dtype != SAD_C128)
      return set_err(ctx, SAD_EINVAL, "complex factors need a complex128 workspace");
    if (!w->pvecs) {
      if (ctx_malloc(ctx, (void**)&w->pvecs, blk * 2) != cudaSuccess)
        return set_err(ctx, SAD_ENOMEM, "BiCGstab preconditioner vectors allocation failed");
      w->bytes += (int64_t)(blk * 2);
    }
    a.phat = w->pvecs;
    a.shat = w->pvecs + blk;
  }
  w->st.tol = tol_col;
  w->st.maxit = maxit;
  a.st = w->st;
  const int gpw = 32 / R;
  // grid-stride kernels: a few blocks per SM keep the finisher's partial
  // reduction short (small blocks are latency-bound)
  const int grid = grid_for(w->n, kWarps * gpw, std::min(w->max_blocks, ctx->nsm * 4));
  const bool cplx = w->dtype == SAD_C128;
  auto vec = [&](int K) {
    return cplx ? bicg_launch_vec_z(K, a, R, grid, s) : bicg_launch_vec_d(K, a, R, grid, s);
  };
  auto spmm = [&](int K) {
    return cplx ? bicg_launch_spmm_z(K, a, R, op->vals_complex, op->sigma_identity, grid, s)
                : bicg_launch_spmm_d(K, a, R, op->vals_complex, op->sigma_identity, grid, s);
  };
  volatile long long* hf = w->hflag_host;
  for (int i = 0; i < 8; ++i) hf[i] = -1;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  k_bi_init<<<1, 32, 0, s>>>(w->st);
  COUNT_LAUNCH(1);
  CK(ctx, cudaMemsetAsync(x, 0, blkb, s));
  CK(ctx, cudaMemcpyAsync(a.r, rhs, blkb, cudaMemcpyDeviceToDevice, s));
  long long cycles = 0;
  const int LAG = 3;
  for (;;) {
    // one run of _bicgstab_column per participating column
    if (vec(BI_START)) return set_err(ctx, SAD_EINVAL, "unsupported block width");
    const long long base = hf[0] < 0 ? 0 : hf[0];
    for (long long step = 0;; ++step) {
      bool stop = false;
      int rc = spin_until(ctx, s, [&] {
        long long done = (hf[0] < 0 ? 0 : hf[0]) - base;
        if (done >= 1 && hf[1] == 0) { stop = true; return true; }
        return step - done <= LAG;
      });
      if (rc) return rc;
      if (stop) break;
      // the first iterations are issued before any flag can say "stop":
      // a run that ends early leaves them as no-ops (gated on the masks)
      if (pc) {
        if (vec(BI_PUPD)) return set_err(ctx, SAD_EINVAL, "unsupported block width");
        if ((rc = sad_pc_apply(pc, R, w->dtype, a.p, (void*)a.phat, 0, s))) return rc;
        if (spmm(BI_SPMM_P) || vec(BI_SUPD))
          return set_err(ctx, SAD_EINVAL, "unsupported block width / value type");
        if ((rc = sad_pc_apply(pc, R, w->dtype, a.s, (void*)a.shat, 0, s))) return rc;
        if (spmm(BI_SPMM_S) || vec(BI_RUPD))
          return set_err(ctx, SAD_EINVAL, "unsupported block width / value type");
      } else if (vec(BI_PUPD) || spmm(BI_SPMM_P) || vec(BI_SUPD) || spmm(BI_SPMM_S) || vec(BI_RUPD))
        return set_err(ctx, SAD_EINVAL, "unsupported block width / value type");
      CKL(ctx);
    }
    vec(BI_XUPD);
    spmm(BI_RESID);
    CKL(ctx);
    ++cycles;
    int rc = spin_until(ctx, s, [&] { return hf[2] >= cycles; });
    if (rc) return rc;
    if (hf[3] == 0) break;
  }
  if (res) CK(ctx, cudaMemcpyAsync(res, a.r, blkb, cudaMemcpyDeviceToDevice, s));
  std::vector<long long> it(R);
  std::vector<double> tn(R);
  CK(ctx, cudaMemcpyAsync(it.data(), w->st.it, R * sizeof(long long), cudaMemcpyDeviceToHost, s));
  CK(ctx, cudaMemcpyAsync(tn.data(), w->st.tnorm, R * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(ctx, cudaStreamSynchronize(s));
  for (int c = 0; c < R; ++c) {
    if (iters_host) iters_host[c] = it[c];
    if (resnorm_host) resnorm_host[c] = tn[c];
    if (conv_host) conv_host[c] = tn[c] <= tol_col ? 1 : 0;
  }
  return SAD_OK;
}

extern "C" int64_t sad_bicg_bytes(const sad_bicg* w) { return w ? w->bytes : -1; }
