/* precond_oracle.c -- TEST INFRASTRUCTURE ONLY (oracle).
 *
 * Plain-C restatement of the reference's incomplete factorisations and
 * triangular solves (/root/reference/pkg/src/sylvadi/precond.py):
 *   oracle_ilu            precond.py:34-125   row-wise (IKJ) ILU, threshold
 *                                             dropping or pattern restriction
 *   oracle_solve_unit_lower   precond.py:129-137
 *   oracle_solve_upper        precond.py:141-149
 *   oracle_solve_lower        precond.py:153-161
 *   oracle_solve_lower_transposed  precond.py:165-173
 * Complex arithmetic is spelled out in real operations in the order numba
 * lowers it (product (ac-bd, ad+bc); quotient by CPython's _Py_c_quot), so
 * the factors are bit-identical to the reference's on the same input
 * (pinned by tests/test_oracle_pin.py against tests/golden/ref_precond.npz).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this; the product never does.  Build: oracle/build_oracle.py
 * (gcc -O2 -ffp-contract=off -shared -fPIC).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double re, im; } cplx;

static cplx c_mul(cplx a, cplx b) {
  cplx z;
  double ac = a.re * b.re, bd = a.im * b.im, ad = a.re * b.im, bc = a.im * b.re;
  z.re = ac - bd;
  z.im = ad + bc;
  return z;
}

static cplx c_sub(cplx a, cplx b) {
  cplx z = {a.re - b.re, a.im - b.im};
  return z;
}

/* CPython's _Py_c_quot, which numba uses for complex128 / complex128 */
static cplx c_div(cplx a, cplx b) {
  cplx z;
  if (fabs(b.re) >= fabs(b.im)) {
    if (b.re == 0.0) { z.re = NAN; z.im = NAN; return z; }
    double ratio = b.im / b.re;
    double denom = b.re + b.im * ratio;
    z.re = (a.re + a.im * ratio) / denom;
    z.im = (a.im - a.re * ratio) / denom;
  } else {
    double ratio = b.re / b.im;
    double denom = b.re * ratio + b.im;
    z.re = (a.re * ratio + a.im) / denom;
    z.im = (a.im * ratio - a.re) / denom;
  }
  return z;
}

static double c_abs(cplx a) { return hypot(a.re, a.im); }

typedef struct {
  long n, lnnz, unnz;
  long *li, *lj;
  cplx* lv;
  long *ui, *uj;
  cplx* uv;
  int status; /* 0 ok, 1 zero pivot */
} ilu_result;

typedef struct { long* idx; cplx* val; long len, cap; } vec;

static void vec_push(vec* v, long j, cplx x) {
  if (v->len == v->cap) {
    v->cap = v->cap ? 2 * v->cap : 1024;
    v->idx = (long*)realloc(v->idx, (size_t)v->cap * sizeof(long));
    v->val = (cplx*)realloc(v->val, (size_t)v->cap * sizeof(cplx));
  }
  v->idx[v->len] = j;
  v->val[v->len] = x;
  v->len++;
}

/* precond.py:34-125.  Row i: scatter, eliminate with the finished rows
 * k = first..i-1 that are occupied (in increasing k, fill joins the scan),
 * drop |l_ik| < tau (threshold kinds), keep U entries >= tau, pivot check. */
ilu_result* oracle_ilu(long n, const long* indptr, const long* indices, const double* data_ri,
                       double droptol, int restrict_pattern) {
  const cplx* data = (const cplx*)data_ri;
  ilu_result* R = (ilu_result*)calloc(1, sizeof(ilu_result));
  cplx* w = (cplx*)calloc((size_t)n, sizeof(cplx));
  char* occupied = (char*)calloc((size_t)n, 1);
  char* in_pattern = (char*)calloc((size_t)n, 1);
  cplx* udiag = (cplx*)calloc((size_t)n, sizeof(cplx));
  vec L = {0, 0, 0, 0}, U = {0, 0, 0, 0};
  R->n = n;
  R->li = (long*)calloc((size_t)n + 1, sizeof(long));
  R->ui = (long*)calloc((size_t)n + 1, sizeof(long));
  const double tiny = 1e-300; /* precond.py:17 */
  for (long i = 0; i < n; ++i) {
    double rownorm = 0.0;
    long first = n;
    for (long p = indptr[i]; p < indptr[i + 1]; ++p) {
      long j = indices[p];
      cplx v = data[p];
      w[j] = v;
      occupied[j] = 1;
      in_pattern[j] = 1;
      rownorm += (v.re * v.re + v.im * v.im);
      if (j < first) first = j;
    }
    const double tau = droptol * sqrt(rownorm);
    for (long k = first; k < i; ++k) {
      if (!occupied[k]) continue;
      cplx lik = c_div(w[k], udiag[k]);
      if (!restrict_pattern && c_abs(lik) < tau) {
        w[k].re = 0.0; w[k].im = 0.0;
        occupied[k] = 0;
        continue;
      }
      w[k] = lik;
      for (long p = R->ui[k] + 1; p < R->ui[k + 1]; ++p) {
        long j = U.idx[p];
        if (restrict_pattern && !in_pattern[j]) continue;
        w[j] = c_sub(w[j], c_mul(lik, U.val[p]));
        occupied[j] = 1;
      }
    }
    cplx piv = w[i];
    if (c_abs(piv) < tiny) {
      R->status = 1;
      break;
    }
    udiag[i] = piv;
    for (long j = first; j < i; ++j)
      if (occupied[j]) vec_push(&L, j, w[j]);
    R->li[i + 1] = L.len;
    vec_push(&U, i, piv);
    for (long j = i + 1; j < n; ++j)
      if (occupied[j] && (restrict_pattern || c_abs(w[j]) >= tau)) vec_push(&U, j, w[j]);
    R->ui[i + 1] = U.len;
    for (long j = first; j < n; ++j) {
      w[j].re = 0.0; w[j].im = 0.0;
      occupied[j] = 0;
      in_pattern[j] = 0;
    }
  }
  R->lnnz = L.len; R->lj = L.idx; R->lv = L.val;
  R->unnz = U.len; R->uj = U.idx; R->uv = U.val;
  free(w); free(occupied); free(in_pattern); free(udiag);
  return R;
}

void oracle_ilu_sizes(const ilu_result* R, long* lnnz, long* unnz, int* status) {
  *lnnz = R->lnnz; *unnz = R->unnz; *status = R->status;
}

void oracle_ilu_copy(const ilu_result* R, long* li, long* lj, double* lv, long* ui, long* uj,
                     double* uv) {
  memcpy(li, R->li, ((size_t)R->n + 1) * sizeof(long));
  memcpy(ui, R->ui, ((size_t)R->n + 1) * sizeof(long));
  if (R->lnnz) {
    memcpy(lj, R->lj, (size_t)R->lnnz * sizeof(long));
    memcpy(lv, R->lv, (size_t)R->lnnz * sizeof(cplx));
  }
  if (R->unnz) {
    memcpy(uj, R->uj, (size_t)R->unnz * sizeof(long));
    memcpy(uv, R->uv, (size_t)R->unnz * sizeof(cplx));
  }
}

void oracle_ilu_free(ilu_result* R) {
  if (!R) return;
  free(R->li); free(R->lj); free(R->lv); free(R->ui); free(R->uj); free(R->uv);
  free(R);
}

/* b: one column, complex interleaved, stride `ld` complex elements between rows */
#define B(i) (b[(size_t)(i) * (size_t)ld])

void oracle_solve_unit_lower(long n, const long* indptr, const long* indices, const double* data_ri,
                             double* b_ri, long ld) {
  const cplx* data = (const cplx*)data_ri;
  cplx* b = (cplx*)b_ri;
  for (long i = 0; i < n; ++i) {
    cplx acc = B(i);
    for (long p = indptr[i]; p < indptr[i + 1]; ++p) acc = c_sub(acc, c_mul(data[p], B(indices[p])));
    B(i) = acc;
  }
}

void oracle_solve_upper(long n, const long* indptr, const long* indices, const double* data_ri,
                        double* b_ri, long ld) {
  const cplx* data = (const cplx*)data_ri;
  cplx* b = (cplx*)b_ri;
  for (long i = n - 1; i >= 0; --i) {
    cplx acc = B(i);
    for (long p = indptr[i] + 1; p < indptr[i + 1]; ++p)
      acc = c_sub(acc, c_mul(data[p], B(indices[p])));
    B(i) = c_div(acc, data[indptr[i]]);
  }
}

void oracle_solve_lower(long n, const long* indptr, const long* indices, const double* data_ri,
                        double* b_ri, long ld) {
  const cplx* data = (const cplx*)data_ri;
  cplx* b = (cplx*)b_ri;
  for (long i = 0; i < n; ++i) {
    cplx acc = B(i);
    for (long p = indptr[i]; p < indptr[i + 1] - 1; ++p)
      acc = c_sub(acc, c_mul(data[p], B(indices[p])));
    B(i) = c_div(acc, data[indptr[i + 1] - 1]);
  }
}

void oracle_solve_lower_transposed(long n, const long* indptr, const long* indices,
                                   const double* data_ri, double* b_ri, long ld) {
  const cplx* data = (const cplx*)data_ri;
  cplx* b = (cplx*)b_ri;
  for (long i = n - 1; i >= 0; --i) {
    B(i) = c_div(B(i), data[indptr[i + 1] - 1]);
    cplx xi = B(i);
    for (long p = indptr[i]; p < indptr[i + 1] - 1; ++p)
      B(indices[p]) = c_sub(B(indices[p]), c_mul(data[p], xi));
  }
}
