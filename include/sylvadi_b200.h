/*
 * sylvadi_b200.h -- C-ABI of the B200-native inner-solve hot path of the
 * inexact low-rank Sylvester ADI method (arXiv 2312.02891).
 *
 * The reference package `sylvadi` (pure Python; /root/reference/pkg/src/sylvadi)
 * reaches native code only through scipy/numpy.  Each entry point below replaces
 * the reference interface cited next to it; the Python host mirror
 * (paper_2312_02891_b200/_lib.py, binding.py, adi.py) binds them with ctypes.
 *
 * Conventions
 *   - Matrices are real CSR: int32 row offsets (n+1), int32 column indices,
 *     float64 values (sparse.py:21-53: canonical, sorted, real).
 *   - Vector blocks are n x r, ROW-MAJOR (element (i,c) at i*r + c), either
 *     float64 (SAD_F64) or interleaved complex128 (SAD_C128).  1 <= r <= 8.
 *   - Pointers named *_dev are device pointers; *_host are host pointers.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Every call returns SAD_OK (0) or an error code; sad_last_error(ctx)
 *     gives the message.  Non-convergence of an inner solve is NOT an error
 *     (conv_host[c] = 0), exactly like the reference (adi.py:597-599).
 *   - The library owns the handles it creates until the matching *_destroy;
 *     the caller owns every buffer it passes in.  No global state; one ctx per
 *     device; calls on one ctx must be serialised by the caller.
 */
#ifndef SYLVADI_B200_H
#define SYLVADI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum sad_status {
  SAD_OK = 0,
  SAD_EINVAL = 1,      /* ValueError / DimensionMismatch (krylov.py:29-35, sparse.py:112-114) */
  SAD_EBREAKDOWN = 2,  /* FactorizationBreakdown: zero Jacobi diagonal (precond.py:274-275) */
  SAD_ECUDA = 3,       /* CUDA runtime failure */
  SAD_ENCCL = 4,       /* reserved for the multi-GPU path */
  SAD_ENOMEM = 5       /* device allocation failed */
};

enum sad_dtype { SAD_F64 = 0, SAD_C128 = 1 };
/* GMRES engines: one cooperative persistent kernel per solve (default), or the
 * multi-kernel CGS2 pipeline (one launch per phase, host-polled). */
enum sad_engine { SAD_ENGINE_MULTI = 0, SAD_ENGINE_PERSISTENT = 1 };
/* sad_gmres_set_option keys */
enum sad_option { SAD_OPT_ENGINE = 0, SAD_OPT_MAX_SMS = 1, SAD_OPT_MIN_ELEMS_PER_THREAD = 2,
                  SAD_OPT_DIRECT_A = 3 /* persistent phase A: -1 auto, 0 TMA ring, 1 direct */,
                  SAD_OPT_RESIDENT_CSR = 4 /* 1 (default): small CSR slabs stay in shared memory */ };
enum sad_precond { SAD_PRECOND_NONE = 0, SAD_PRECOND_JACOBI = 1 };

typedef struct sad_ctx sad_ctx;
typedef struct sad_csr sad_csr;
typedef struct sad_op sad_op;
typedef struct sad_gmres sad_gmres;

/* ABI version (bumped on any signature change). */
int sad_version(void);
/* Number of CUDA kernels this library has launched in the process (evidence
 * that the device path ran; bench.py reports it as gpu_launches). */
int64_t sad_kernel_launches(void);

/* Context bound to one CUDA device. */
int sad_ctx_create(int device, sad_ctx** out);
int sad_ctx_destroy(sad_ctx* ctx);
const char* sad_last_error(const sad_ctx* ctx);
/* Number of SMs of the context's device (grid sizing is a multiple of it). */
int sad_ctx_num_sms(const sad_ctx* ctx);

/*
 * Upload a real CSR matrix (host arrays).  Replaces SparseMatrix (sparse.py:21-100).
 * build_transpose != 0 also stores the explicit transpose as CSR so adjoint
 * products are deterministic row gathers (replaces the CSC scatter of
 * spmv_transpose, sparse.py:128-135).
 */
int sad_csr_create(sad_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz,
                   const int32_t* rowptr_host, const int32_t* colidx_host,
                   const double* vals_host, int build_transpose, sad_csr** out);
int sad_csr_destroy(sad_csr* csr);
int64_t sad_csr_nnz(const sad_csr* csr);

/*
 * Shifted operator Op = base + sigma*mass (mass NULL = identity) or, with
 * adjoint != 0, Op = base^T + conj(sigma) mass^T.  Replaces ShiftedOperator
 * (sparse.py:158-206) plus the Jacobi factorisation of its assembled form
 * (precond.py:272-276, adi.py:454-466): precond_kind SAD_PRECOND_JACOBI builds
 * dinv = 1/diag(Op) on device and returns SAD_EBREAKDOWN if |diag| < 1e-300.
 */
int sad_op_create(sad_ctx* ctx, const sad_csr* base, const sad_csr* mass,
                  double sigma_re, double sigma_im, int adjoint,
                  int precond_kind, sad_op** out);
int sad_op_destroy(sad_op* op);
/* Copy dinv (n complex128 values, interleaved) to host; for tests. */
int sad_op_get_dinv(const sad_op* op, double* dinv_host);

/* y = Op x  (ShiftedOperator.apply, sparse.py:192-206). */
int sad_op_apply(sad_op* op, int r, int dtype, const void* x_dev, void* y_dev,
                 void* stream);
/* y = b - Op x  (the true residual, krylov.py:62). */
int sad_op_residual(sad_op* op, int r, int dtype, const void* b_dev,
                    const void* x_dev, void* y_dev, void* stream);
/* y = A x or y = A^T x for a plain CSR (spmv / spmv_transpose, sparse.py:118-135;
 * transpose needs build_transpose at creation). */
int sad_csr_apply(sad_csr* csr, int transpose, int r, int dtype,
                  const void* x_dev, void* y_dev, void* stream);

/*
 * Krylov workspace for Jacobi-right-preconditioned GMRES(restart) or
 * FGMRES(restart) on n x r blocks (SURVEY.md 8a "Algorithm contract for a8").
 * Holds the (restart+1) basis blocks (plus restart Z blocks when flexible).
 */
int sad_gmres_create(sad_ctx* ctx, int64_t n, int r, int dtype, int restart,
                     int flexible, sad_gmres** out);
int sad_gmres_destroy(sad_gmres* ws);
/* Device bytes held by the workspace. */
int64_t sad_gmres_bytes(const sad_gmres* ws);
/* Engine / grid options (see enum sad_option).  SAD_OPT_MAX_SMS caps the SMs a
 * persistent solve occupies so that the A- and B-side solves can be resident
 * at the same time on two streams (0 = all SMs). */
int sad_gmres_set_option(sad_gmres* ws, int key, int value);

/*
 * Solve Op X = RHS column by column (batched in lock-step) to the per-column
 * absolute target tol_col = delta / r (krylov.py:164).  Replaces
 * bicgstab(InnerSolveRequest(...)) (krylov.py:17-38,160-184) behind
 * SolverBinding.solve (adi.py:473-488).
 *   rhs_dev   n x r block (dtype of the workspace)
 *   x_dev     n x r solution (overwritten; zero initial guess)
 *   res_dev   n x r true residual RHS - Op X after termination, or NULL
 *   maxit     per-column iteration cap (max_iterations, adi.py:142)
 *   iters_host[r]   Arnoldi steps per column (int64)
 *   resnorm_host[r] ||res(:,c)||_2
 *   conv_host[r]    resnorm <= tol_col
 * The host synchronises only at the restart-cycle boundaries.
 */
int sad_gmres_solve(sad_gmres* ws, sad_op* op, const void* rhs_dev, void* x_dev,
                    void* res_dev, double tol_col, int maxit, void* stream,
                    int64_t* iters_host, double* resnorm_host,
                    uint8_t* conv_host);

/*
 * The same solve split in two: sad_gmres_launch enqueues it on `stream` and
 * returns (persistent engine; the multi-kernel engine runs to completion
 * inside launch); sad_gmres_finish waits and fills the result arrays.  Lets
 * one host thread keep the A- and B-side solves in flight together.
 */
int sad_gmres_launch(sad_gmres* ws, sad_op* op, const void* rhs_dev, void* x_dev,
                     double tol_col, int maxit, void* stream);
int sad_gmres_finish(sad_gmres* ws, void* res_dev, void* stream, int64_t* iters_host,
                     double* resnorm_host, uint8_t* conv_host);

/*
 * Same solve, but a fixed number of Arnoldi steps (no stopping test inside the
 * cycle; config 4 "100 fixed block-GMRES iterations").  When timing_ms_host is
 * not NULL it receives (CUDA events on `stream`):
 *   multi-kernel engine: {spmm_ms, orth_ms, cycle_end_ms, initial_residual_ms}
 *   persistent engine:   {kernel_ms, phaseA_ms, phaseC_ms, algorithmic_bytes}
 */
int sad_gmres_fixed(sad_gmres* ws, sad_op* op, const void* rhs_dev, void* x_dev,
                    void* res_dev, int steps, void* stream,
                    double* resnorm_host, double* timing_ms_host);

/*
 * Profiling of sad_gmres_solve: enable=1 resets the counters; enable=0 stops.
 * stats_host[13] (may be NULL) receives the counters accumulated so far.
 * Multi-kernel engine (synchronous stepping with CUDA events):
 *   {spmm_ms, spmm_launches, spmm_algorithmic_bytes, orth_ms, arnoldi_steps,
 *    orth_bytes, cycle_end_ms, cycles}
 * Persistent engine (CUDA events around each cooperative launch, phase times
 * from %globaltimer in block 0):
 *   {kernel_ms, launches, algorithmic_bytes, phaseA_ms (SpMM + basis dots),
 *    arnoldi_steps, phaseC_ms (basis update), cycle_end_ms, cycles,
 *    workA_ms, workC_ms (block 0 before the barrier), finA_ms, finC_ms (the
 *    reducing block's serial section), spmmA_ms (block 0 inside the phase-A SpMM)}
 */
int sad_gmres_profile(sad_gmres* ws, int enable, double* stats_host);

/* G = X^H Y for n x r blocks (r x r, complex128 interleaved, row a col b =
 * sum_i conj(X[i,a]) Y[i,b]); written to host.  Feeds block_norm,
 * block_residual_norm and computed_residual_norm (adi.py:54-70, krylov.py:53-58). */
int sad_gram(sad_ctx* ctx, int64_t n, int r, int dtype, const void* x_dev,
             const void* y_dev, double* gram_host, void* stream);

/* y += a * x on n x r blocks (complex a; for SAD_F64 a_im must be 0). */
int sad_axpy(sad_ctx* ctx, int64_t n, int r, int dtype, double a_re, double a_im,
             const void* x_dev, void* y_dev, void* stream);

/*
 * Fused ADI step epilogue (adi.py:518-530) on device blocks, one launch:
 *   w += gamma * mz ;  t += conj(gamma) * cty
 * and the six r x r Gram matrices the host tolerance logic needs, written to
 * gram_host[6][r][r] (complex128): resA^H resA, resB^H resB, mz^H mz,
 * cty^H cty, w^H w (updated), t^H t (updated).  nA/nB rows on the A/B side.
 */
int sad_adi_epilogue(sad_ctx* ctx, int64_t nA, int64_t nB, int r, int dtype,
                     double gamma_re, double gamma_im, const void* mz_dev,
                     const void* resA_dev, void* w_dev, const void* cty_dev,
                     const void* resB_dev, void* t_dev, double* gram_host,
                     void* stream);

/*
 * Tall-skinny products over a low-rank factor X (n x K, row-major, leading
 * dimension ldx >= K, F64 or C128) for the verification diagnostics: the
 * power iteration of true_residual_norm (adi.py:682-726) evaluates
 * `Y.conj().T @ x` and `Z @ c` (adi.py:692-705) with these.
 *   sad_ts_hgemv: out_host[K][nvec] = X^H V   (V: n x nvec complex128 device
 *                 block, nvec in {1, 2}; deterministic block-ordered sums)
 *   sad_ts_gemv:  Y[n][nvec] (+)= X C        (C_host: K x nvec complex128;
 *                 accumulate != 0 adds to Y; Y complex128 device block)
 */
int sad_ts_hgemv(sad_ctx* ctx, int64_t n, int64_t K, int64_t ldx, int xdtype, const void* x_dev,
                 int nvec, const void* v_dev, double* out_host, void* stream);
int sad_ts_gemv(sad_ctx* ctx, int64_t n, int64_t K, int64_t ldx, int xdtype, const void* x_dev,
                int nvec, const double* c_host, void* y_dev, int accumulate, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SYLVADI_B200_H */
