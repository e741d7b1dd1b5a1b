// sad_precond.cuh -- sparse triangular solves for the reference's incomplete-
// factorisation preconditioners (precond.py:129-173, applied by
// IncompleteFactorization.apply / apply_spd, precond.py:208-256) on n x R blocks.
//
// One kernel covers the four solves: the host stores every factor as
// "off-diagonal entries in the order the reference subtracts them" + an optional
// diagonal (unit-lower L: none; U: its first entry; G: its last entry; G^T: the
// transposed rows with descending column order, which is the order the
// reference's scatter solve updates b[i]), so row i is
//     x_i = (b_i - sum_p v_p x_{col_p}) / d_i        (sum taken in order, p ascending)
// with every product and difference rounded once (no fma) and the complex
// quotient by the algorithm numba uses (CPython's _Py_c_quot): the result is
// bit-identical to the reference's for the same factor.
//
// Parallelism: rows are sorted by dependency level on the host; a warp takes
// the next task (32/R rows of ONE level, a group of R lanes per row, lane c of
// a group = column c) from an atomic ticket and each lane waits for the
// elements it reads.  Every solved element is published as 16-byte cells
// {value, epoch tag} written with ONE 128-bit store and polled with ONE 128-bit
// load (a complex element is two cells, real and imaginary part, each with its
// tag): value and flag travel together, so a level costs one L2 round trip
// instead of three (flag poll, then the data load, after a release store) --
// the flag-array version ran at 2.6 us per level.  Tickets are handed out in level order, so a warp only ever waits on
// rows whose warps are already running or done: no deadlock, no grid barrier,
// one launch per triangular solve.  The chain of levels is latency-bound
// (about one L2 round trip per level), which is inherent to these
// preconditioners -- the hot path's preconditioner is Jacobi.
#pragma once

#include "sad_kernels.cuh"

namespace sad {

struct TriArgs {
  long long n;
  const int* rowptr;
  const int* colidx;
  const void* vals;     // VT, off-diagonal entries
  const void* diag;     // VT [n] or nullptr (unit diagonal)
  const int* order;     // [ntasks * (32/R)] rows by level, -1 = padding
  int ntasks;
  void* cells;          // [n * R] (x 2 for complex blocks) 16-byte {value, epoch} cells
  long long epoch;
  unsigned* counter;    // task ticket (zeroed before the launch)
  const void* b;        // XT, n x R
  void* x;              // XT, n x R (may alias b)
  int negate;           // solve for -b (the sign of a negated Cholesky process)
};

// single-rounding arithmetic in the reference's operation order
__device__ __forceinline__ double tmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double2 tmul(double a, double2 b) {
  return make_double2(__dmul_rn(a, b.x), __dmul_rn(a, b.y));
}
__device__ __forceinline__ double2 tmul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double tsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double2 tsub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double tdiv(double a, double d) { return __ddiv_rn(a, d); }
__device__ __forceinline__ double2 tdiv(double2 a, double d) {
  return make_double2(__ddiv_rn(a.x, d), __ddiv_rn(a.y, d));
}
__device__ __forceinline__ double2 tdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double ratio = __ddiv_rn(b.y, b.x);
    const double denom = __dadd_rn(b.x, __dmul_rn(b.y, ratio));
    return make_double2(__ddiv_rn(__dadd_rn(a.x, __dmul_rn(a.y, ratio)), denom),
                        __ddiv_rn(__dsub_rn(a.y, __dmul_rn(a.x, ratio)), denom));
  }
  const double ratio = __ddiv_rn(b.x, b.y);
  const double denom = __dadd_rn(__dmul_rn(b.x, ratio), b.y);
  return make_double2(__ddiv_rn(__dadd_rn(__dmul_rn(a.x, ratio), a.y), denom),
                      __ddiv_rn(__dsub_rn(__dmul_rn(a.y, ratio), a.x), denom));
}
__device__ __forceinline__ double tneg(double a) { return -a; }
__device__ __forceinline__ double2 tneg(double2 a) { return make_double2(-a.x, -a.y); }

// One cell is read and written as a single .b128 access (single-copy atomic:
// value and tag can never be seen torn).
struct __align__(16) TriCell { double v; long long tag; };

__device__ __forceinline__ TriCell ld_cell(const TriCell* p) {
  TriCell c;
  unsigned long long lo, hi;
  asm volatile("{\n\t.reg .b128 q;\n\tld.relaxed.gpu.global.b128 q, [%2];\n\tmov.b128 {%0, %1}, q;\n\t}"
               : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
  c.v = __longlong_as_double((long long)lo);
  c.tag = (long long)hi;
  return c;
}
__device__ __forceinline__ void st_cell(TriCell* p, double v, long long tag) {
  asm volatile("{\n\t.reg .b128 q;\n\tmov.b128 q, {%1, %2};\n\tst.relaxed.gpu.global.b128 [%0], q;\n\t}" ::"l"(p),
               "l"((unsigned long long)__double_as_longlong(v)), "l"((unsigned long long)tag)
               : "memory");
}
// wait for element d of epoch `ep` and return it
__device__ __forceinline__ double tri_wait(const TriCell* cells, size_t d, long long ep, double) {
  TriCell c;
  do { c = ld_cell(cells + d); } while (c.tag != ep);
  return c.v;
}
__device__ __forceinline__ double2 tri_wait(const TriCell* cells, size_t d, long long ep, double2) {
  TriCell re, im;
  do { re = ld_cell(cells + 2 * d); } while (re.tag != ep);
  do { im = ld_cell(cells + 2 * d + 1); } while (im.tag != ep);
  return make_double2(re.v, im.v);
}
__device__ __forceinline__ void tri_publish(TriCell* cells, size_t e, long long ep, double v) {
  st_cell(cells + e, v, ep);
}
__device__ __forceinline__ void tri_publish(TriCell* cells, size_t e, long long ep, double2 v) {
  st_cell(cells + 2 * e, v.x, ep);
  st_cell(cells + 2 * e + 1, v.y, ep);
}

template <typename XT, typename VT, int R>
__global__ void __launch_bounds__(kThreads) k_sptrsv(TriArgs a) {
  constexpr int GPW = 32 / R;
  const int lane = threadIdx.x & 31;
  const int grp = lane / R, c = lane - grp * R;
  const bool lane_ok = grp < GPW;
  const VT* vals = reinterpret_cast<const VT*>(a.vals);
  const VT* diag = reinterpret_cast<const VT*>(a.diag);
  const XT* b = reinterpret_cast<const XT*>(a.b);
  XT* x = reinterpret_cast<XT*>(a.x);
  TriCell* cells = reinterpret_cast<TriCell*>(a.cells);
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(a.counter, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= (unsigned)a.ntasks) break;
    const int row = lane_ok ? __ldg(a.order + (size_t)t * GPW + grp) : -1;
    if (row >= 0) {
      const size_t e = (size_t)row * R + c;
      XT acc = b[e];
      if (a.negate) acc = tneg(acc);
      const int p1 = __ldg(a.rowptr + row + 1);
      for (int p = __ldg(a.rowptr + row); p < p1; ++p) {
        const int col = __ldg(a.colidx + p);
        const VT v = __ldg(vals + p);
        const size_t d = (size_t)col * R + c;
        acc = tsub(acc, tmul(v, tri_wait(cells, d, a.epoch, XT())));
      }
      if (diag) acc = tdiv(acc, __ldg(diag + row));
      tri_publish(cells, e, a.epoch, acc);    // for the rows that depend on this one
      x[e] = acc;                             // the result block
    }
  }
}

}  // namespace sad
