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
  SAD_ENCCL = 4,       /* NCCL missing or a collective failed (row-partitioned solves) */
  SAD_ENOMEM = 5       /* device allocation failed */
};

enum sad_dtype { SAD_F64 = 0, SAD_C128 = 1 };
/* GMRES engines: one cooperative persistent kernel per solve (default), or the
 * multi-kernel CGS2 pipeline (one launch per phase, host-polled). */
enum sad_engine { SAD_ENGINE_MULTI = 0, SAD_ENGINE_PERSISTENT = 1 };
/* sad_gmres_set_option keys */
enum sad_option { SAD_OPT_ENGINE = 0, SAD_OPT_MAX_SMS = 1, SAD_OPT_MIN_ELEMS_PER_THREAD = 2,
                  SAD_OPT_DIRECT_A = 3 /* persistent phase A: -1 auto, 0 TMA ring, 1 direct */,
                  SAD_OPT_RESIDENT_CSR = 4, /* 1 (default): small CSR slabs stay in shared memory */
                  SAD_OPT_DIST_ORTH = 5, /* row-partitioned: 1 (default) delayed-Gram CGS2, 0 CGS2 */
                  SAD_OPT_DEBUG_DELAY = 6 /* tests: the persistent kernel's last block idles this
                                             many ns after every phase-C barrier (race stress) */ };
/* precond.py:15 KINDS.  NONE / JACOBI are folded into the operator (sad_op_create);
 * the incomplete factorisations are separate handles (sad_pc_create). */
enum sad_precond { SAD_PRECOND_NONE = 0, SAD_PRECOND_JACOBI = 1, SAD_PRECOND_ILU0 = 2,
                   SAD_PRECOND_ILUT = 3, SAD_PRECOND_IC0 = 4, SAD_PRECOND_ICT = 5 };

typedef struct sad_ctx sad_ctx;
typedef struct sad_csr sad_csr;
typedef struct sad_op sad_op;
typedef struct sad_gmres sad_gmres;
typedef struct sad_comm sad_comm;
typedef struct sad_halo sad_halo;
typedef struct sad_bicg sad_bicg;
typedef struct sad_minres sad_minres;
typedef struct sad_pc sad_pc;

/* ABI version (bumped on any signature change). */
int sad_version(void);
/* Number of CUDA kernels this library has launched in the process (evidence
 * that the device path ran; bench.py reports it as gpu_launches). */
int64_t sad_kernel_launches(void);

/* Context bound to one CUDA device. */
int sad_ctx_create(int device, sad_ctx** out);
int sad_ctx_destroy(sad_ctx* ctx);
const char* sad_last_error(const sad_ctx* ctx);
/* Release the device memory the context caches for reuse (buffers of
 * destroyed matrices, operators and workspaces; see sad_capi.cu DevCache). */
int sad_ctx_trim(sad_ctx* ctx);
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
/* The banded SpMM plan of the operator's sparsity pattern, if it has one
 * (built at creation for operators with >= 2^20 nonzeros, or as the environment
 * variable SAD_SPMM_BAND = 0 / 1 says): rows in tiles, the x rows a tile
 * reads staged in shared memory by TMA, 16-bit local column indices.  info[7] =
 * plan present (0/1), tiles, padded entries, nonzeros, local x rows per tile
 * (max), padded row length (max), rows per tile (256, 128 or 64; SAD_BAND_ROWS
 * overrides).  Patterns that do not fit run the CSR kernels.  Plans are built
 * on first use, per class: 0 = the stand-alone SpMM (sad_op_apply / residual,
 * the multi-kernel engine), 1 = the SpMM sub-phase of the persistent GMRES
 * kernel (smaller tiles, SAD_BAND_ROWS_P). */
int sad_op_band_info(sad_op* op, int plan_class, int64_t* info);
int sad_op_get_dinv(const sad_op* op, double* dinv_host);

/* y = Op x  (ShiftedOperator.apply, sparse.py:192-206). */
int sad_op_apply(sad_op* op, int r, int dtype, const void* x_dev, void* y_dev,
                 void* stream);
/*
 * y = Op x between HOST buffers (x_host, y_host: n x r row-major), the
 * reference-facing form of ShiftedOperator.apply (sparse.py:192-206), which
 * takes and returns host numpy blocks.  Returns when y_host is filled.  The
 * block moves in row chunks: uploads on one stream, the SpMM of an output chunk
 * as soon as the x rows it reads have landed, downloads on a third stream
 * (both PCIe directions and the SpMM overlap when the buffers are pinned).
 * Device staging is owned by the operator and reused across calls.
 */
int sad_op_apply_host(sad_op* op, int r, int dtype, const void* x_host, void* y_host,
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
 * not NULL (8 doubles) it receives (CUDA events on `stream`):
 *   multi-kernel engine: {spmm_ms, orth_ms, cycle_end_ms, initial_residual_ms}
 *   persistent engine:   {kernel_ms, phaseA_ms, phaseC_ms, algorithmic_bytes,
 *                         spmmA_ms, cycle_end_ms, arnoldi_steps, 0}
 *   (phase times: block 0's %globaltimer; spmmA = its SpMM sub-phase of phase A)
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

/* ---------------------------------------------------------------------------
 * Row-partitioned inner solves (one operator split into
 * contiguous row slabs, halo exchange before every SpMM, all-reduce of every
 * block dot; Hessenberg, Givens and masks replicated on every rank).  The
 * reference has no multi-process path: these extend SolverBinding.solve
 * (adi.py:473-488) to a slab of the operator; the Python mirror is
 * paper_2312_02891_b200/rowpart.py.
 *
 * Communicators: NCCL (one process per GPU; sad_comm_unique_id on rank 0, the
 * 128 bytes broadcast by the caller, sad_comm_create_nccl on every rank;
 * libnccl.so.2 is bound with dlopen), or an in-process group of `nranks` ranks
 * on one device (sad_comm_create_local) whose kernels run in rank order with
 * a device sum for the all-reduce and device copies for send/recv.
 * Every sad_dist_* call takes `nl` local ranks: 1 for NCCL, nranks for a group;
 * per-rank arguments are arrays of length nl.
 * ------------------------------------------------------------------------- */
int sad_comm_unique_id(uint8_t* id_out /* 128 bytes */);
const char* sad_comm_nccl_error(void);
int sad_comm_create_nccl(sad_ctx* ctx, int nranks, int rank, const uint8_t* id, sad_comm** out);
int sad_comm_create_local(sad_ctx* ctx, int nranks, sad_comm** out);
int sad_comm_destroy(sad_comm* comm);
int sad_comm_size(const sad_comm* comm);
int sad_comm_local_ranks(const sad_comm* comm);

/* Halo plan of one rank: rows [0, n_loc) are local, [n_loc, n_loc + n_halo)
 * the halo, grouped by owning rank q at recv_off[q] .. recv_off[q+1];
 * send_rows[send_off[q] .. send_off[q+1]) are the local rows rank q needs. */
int sad_halo_create(sad_ctx* ctx, int nranks, int rank, int64_t n_loc, int64_t n_halo,
                    const int64_t* send_off, const int32_t* send_rows, const int64_t* recv_off,
                    sad_halo** out);
int sad_halo_destroy(sad_halo* halo);

/* Local slab CSR, columns remapped to [local | halo] in the global matrix's
 * per-row order (not increasing after the remap; no transpose is built). */
int sad_local_csr_create(sad_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz,
                         const int32_t* rowptr, const int32_t* colidx, const double* vals,
                         sad_csr** out);
/* Op = slab + sigma I (the B side passes the slab of B^T and conj(sigma));
 * Jacobi dinv over [local | halo], the halo part filled by sad_dist_op_setup. */
int sad_local_op_create(sad_ctx* ctx, const sad_csr* slab, double sre, double sim,
                        int precond_kind, sad_op** out);
int sad_dist_op_setup(sad_comm* comm, int nl, sad_op* const* ops, sad_halo* const* halos,
                      void* stream);
/* halo rows of n_ext-row blocks; y = Op x (x_ext's halo rows are overwritten) */
int sad_dist_halo_exchange(sad_comm* comm, int nl, sad_halo* const* halos, void* const* blocks,
                           int r, int dtype, void* stream);
int sad_dist_op_apply(sad_comm* comm, int nl, sad_op* const* ops, sad_halo* const* halos, int r,
                      int dtype, void* const* x_ext, void* const* y, void* stream);
/* in-place sum over the ranks of `count` doubles per rank buffer */
int sad_dist_allreduce(sad_comm* comm, int nl, double* const* bufs, int64_t count, void* stream);
/* workspace of one rank: basis blocks of n_ext rows (the halo travels with them) */
int sad_dist_gmres_create(sad_ctx* ctx, int64_t n_loc, int64_t n_ext, int r, int dtype,
                          int restart, int flexible, sad_gmres** out);
/* sad_gmres_solve on a row-partitioned operator: rhs/x/res are n_loc x r
 * slabs per local rank; iters/resnorm/conv are replicated (filled once). */
int sad_dist_gmres_solve(sad_comm* comm, int nl, sad_gmres* const* ws, sad_op* const* ops,
                         sad_halo* const* halos, const void* const* rhs_dev, void* const* x_dev,
                         void* const* res_dev, double tol_col, int maxit, void* stream,
                         int64_t* iters_host, double* resnorm_host, uint8_t* conv_host);

/* ---------------------------------------------------------------------------
 * The reference's own inner solver on the device: right-preconditioned
 * BiCGstab per column with the drift-resume loop (krylov.py:82-184), batched
 * over the r columns of a block (each column an independent run, advancing in
 * lock step; scalars, breakdown restarts and stopping on the device).
 * Replaces bicgstab(InnerSolveRequest(op, rhs, tol, maxit, precond))
 * (krylov.py:160) behind SolverBinding.solve (adi.py:473-488): same stopping
 * rule (recurrence residual <= tol_col, then the true residual with resume),
 * iteration counts per column, residual = b - Op x.
 * ------------------------------------------------------------------------- */
int sad_bicg_create(sad_ctx* ctx, int64_t n, int r, int dtype, sad_bicg** out);
int sad_bicg_destroy(sad_bicg* ws);
int64_t sad_bicg_bytes(const sad_bicg* ws);
int sad_bicg_solve(sad_bicg* ws, sad_op* op, const void* rhs_dev, void* x_dev, void* res_dev,
                   double tol_col, int maxit, void* stream, int64_t* iters_host,
                   double* resnorm_host, uint8_t* conv_host);

/* ---------------------------------------------------------------------------
 * The reference's inner solver for Hermitian sides on the device: split-
 * preconditioned MINRES (Paige-Saunders) per column (krylov.py:187-287),
 * batched over the r columns of a block in lock step, the recurrence scalars,
 * true-residual checks and stopping on the device.  Replaces
 * minres(InnerSolveRequest(op, rhs, tol, maxit, precond)) (krylov.py:271)
 * behind SolverBinding.solve when uses_minres(shift) (adi.py:468-488): real
 * shift, symmetric base/mass, preconditioner "none" or "jacobi" (SPD split
 * |dinv|, precond.py:242-256).  Same stopping rule (phibar <= check_at, then
 * ||b - Op x|| <= tol_col), iteration counts per column, residual = b - Op x.
 * SAD_EINVAL for a complex shift; SAD_EBREAKDOWN if beta1^2 <= 0
 * (the reference's RuntimeError, krylov.py:203-205).
 * ------------------------------------------------------------------------- */
int sad_minres_create(sad_ctx* ctx, int64_t n, int r, int dtype, sad_minres** out);
int sad_minres_destroy(sad_minres* ws);
int64_t sad_minres_bytes(const sad_minres* ws);
int sad_minres_solve(sad_minres* ws, sad_op* op, const void* rhs_dev, void* x_dev,
                     void* res_dev, double tol_col, int maxit, void* stream,
                     int64_t* iters_host, double* resnorm_host, uint8_t* conv_host);

/* ---------------------------------------------------------------------------
 * Incomplete-factorisation preconditioners (the paper's iLU / iC(., 0.1),
 * PAPER.md:638-649).  sad_pc_create replaces factorize(op.assembled(), kind,
 * droptol, shift) (precond.py:307-357) as called by SolverBinding._factorization
 * (adi.py:453-466): the assembled shifted matrix base + shift*mass (mass NULL =
 * identity; conjugate-transposed when adjoint), the row-wise IKJ incomplete LU
 * with threshold dropping (ILUT / ICT: |l_ik| < droptol * ||row||_2 dropped,
 * U entries kept when >= it) or restricted to the matrix pattern (ILU0 / IC0)
 * (precond.py:34-125) and, for the Cholesky kinds, the negation of a negative
 * definite matrix and the fold G = L sqrt(D) (precond.py:279-304, 338-346).
 * The factorisation is computed once per shift on the host (a sequential
 * recurrence with a data-dependent pattern), bit-identical to the reference's;
 * the triangular solves run on the device.  SAD_EBREAKDOWN = the reference's
 * FactorizationBreakdown (zero pivot, or not positive definite up to dropping).
 *
 * sad_pc_apply: y = M^-1 x, IncompleteFactorization.apply (precond.py:224-240,
 * including the sign of a negated Cholesky process); spd != 0: apply_spd
 * (precond.py:242-256), (G G^H)^-1 x, Cholesky kinds only.  y may alias x.
 * One handle serves one stream at a time.
 * sad_pc_info: info[8] = kind, n, nnz of L (or G), nnz of U (0 for Cholesky),
 * complex factors (0/1), dependency levels of the first and second triangular
 * solve, sign.  sad_pc_get_factor: the reference's raw triplets (which = 0: L
 * without its unit diagonal, or G with the diagonal last in each row; which = 1:
 * U with the diagonal first), data interleaved complex128.
 * sad_bicg_solve_pc / sad_minres_solve_pc: the solvers above with the
 * preconditioner argument of InnerSolveRequest (krylov.py:23) given as a handle
 * (NULL = the operator's own none / Jacobi); the operator passed with a BiCGstab
 * handle must be created with SAD_PRECOND_NONE.
 * ------------------------------------------------------------------------- */
int sad_pc_create(sad_ctx* ctx, const sad_csr* base, const sad_csr* mass, double shift_re,
                  double shift_im, int adjoint, int kind, double droptol, sad_pc** out);
int sad_pc_destroy(sad_pc* pc);
int sad_pc_info(const sad_pc* pc, int64_t* info);
int sad_pc_get_factor(const sad_pc* pc, int which, int64_t* indptr, int64_t* indices,
                      double* data_ri);
int sad_pc_apply(sad_pc* pc, int r, int dtype, const void* x_dev, void* y_dev, int spd,
                 void* stream);
int sad_bicg_solve_pc(sad_bicg* ws, sad_op* op, sad_pc* pc, const void* rhs_dev, void* x_dev,
                      void* res_dev, double tol_col, int maxit, void* stream, int64_t* iters_host,
                      double* resnorm_host, uint8_t* conv_host);
int sad_minres_solve_pc(sad_minres* ws, sad_op* op, sad_pc* pc, const void* rhs_dev, void* x_dev,
                        void* res_dev, double tol_col, int maxit, void* stream,
                        int64_t* iters_host, double* resnorm_host, uint8_t* conv_host);

/* ---------------------------------------------------------------------------
 * The device-resident ADI outer loop in native code: run_with_state
 * (adi.py:553-607) with adi_step (adi.py:510-537) for the iterative
 * strategies, inner solves by the persistent GMRES kernel.  Same loop as
 * paper_2312_02891_b200/adi.py DeviceAdi.run, without interpreter overhead per
 * step.  Host scalars as in AdiConfig (adi.py:130-180).
 * ------------------------------------------------------------------------- */
enum sad_strategy { SAD_STRAT_FIXED = 0, SAD_STRAT_DYNAMIC_MID = 1, SAD_STRAT_DYNAMIC_MID_BL = 2,
                    SAD_STRAT_DYNAMIC_B = 3, SAD_STRAT_DYNAMIC_B_BL = 4 };
typedef struct {
  int strategy;                /* enum sad_strategy */
  int kmax;
  int max_inner_iterations;
  double outer_tolerance;
  double xi;
  double gap_budget;           /* used when has_gap_budget != 0 */
  double fixed_delta;
  double delta_min_A, delta_max_A, delta_min_B, delta_max_B;
  int has_gap_budget;          /* 0: AdiConfig.gap_budget is None -> outer_tolerance * ||f g^*||
                                  (adi.py:563-565); a budget of 0.0 is a budget */
} sad_adi_config;
/* records[k][14] per step: scaled_res, delta_A, delta_B, achieved_rA,
 * achieved_rB, inner_it_A, inner_it_B, u, v, a_converged, b_converged,
 * clamped_A_min, clamped_B_min, wall_ms (StepRecord, adi.py:193-210);
 * summary[5]: ||f g^*||, converged, final scaled residual, u, v.
 * opsA/opsB/gammas: per step k (kmax entries; gammas complex interleaved);
 * z_base/y_base: kmax contiguous n x r blocks (z_k, y_k); w, t: f, g in,
 * updated in place; M, C may be NULL (identity; C applied transposed). */
#define SAD_ADI_REC 14
int sad_adi_run(sad_ctx* ctx, const sad_adi_config* cfg, int r, int dtype, int64_t nA, int64_t nB,
                sad_gmres* wsA, sad_gmres* wsB, sad_op* const* opsA, sad_op* const* opsB,
                const double* gammas, sad_csr* M, sad_csr* C, void* w_dev, void* t_dev,
                void* z_base, void* y_base, void* resA_dev, void* resB_dev, void* mz_buf,
                void* cty_buf, int concurrent, void* stream_main, void* streamA, void* streamB,
                double* records, int* steps_out, double* summary);

#ifdef __cplusplus
}
#endif

#endif /* SYLVADI_B200_H */
