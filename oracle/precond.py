"""CPU ORACLE for the reference's incomplete-factorisation preconditioners.

TEST INFRASTRUCTURE ONLY (same rules as oracle/sylvadi_oracle.py: only tests/,
smoke() and bench.py's cpu_baseline leg may import this).

Restates /root/reference/pkg/src/sylvadi/precond.py: the factorisation kernel
and the four triangular solves live in oracle/precond_oracle.c (plain C, built
by oracle/build_oracle.py); this module is the reference's host logic around
them -- ``factorize`` (precond.py:307-357), the Cholesky fold
(precond.py:279-304), ``apply`` / ``apply_spd`` (precond.py:224-256) and the
assembled shifted matrix they are computed from (sparse.py:138-155, 183-190).

Pinned to the reference's own factors and actions, bit for bit, by
tests/test_oracle_pin.py against tests/golden/ref_precond.npz (written by
tests/golden/make_golden_precond.py, which runs the reference).
"""

import ctypes as C
import os

import numpy as np
import scipy.sparse as sp

from . import build_oracle

KINDS = ("none", "jacobi", "ilu0", "ilut", "ic0", "ict")
PIVOT_TINY = 1e-300   # precond.py:17


class FactorizationBreakdown(RuntimeError):
    """precond.py:20-21"""


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = build_oracle.OUT
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(build_oracle.SRC):
            build_oracle.build()
        lib = C.CDLL(path)
        P = C.c_void_p
        lib.oracle_ilu.restype = P
        lib.oracle_ilu.argtypes = [C.c_long, P, P, P, C.c_double, C.c_int]
        lib.oracle_ilu_sizes.argtypes = [P, C.POINTER(C.c_long), C.POINTER(C.c_long),
                                         C.POINTER(C.c_int)]
        lib.oracle_ilu_copy.argtypes = [P] * 7
        lib.oracle_ilu_free.argtypes = [P]
        for name in ("oracle_solve_unit_lower", "oracle_solve_upper", "oracle_solve_lower",
                     "oracle_solve_lower_transposed"):
            getattr(lib, name).argtypes = [C.c_long, P, P, P, P, C.c_long]
        _LIB = lib
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def ilu_kernel(n, indptr, indices, data, droptol, restrict_pattern):
    """precond.py:34-125 -> (li, lj, lv, ui, uj, uv, status)."""
    lib = _lib()
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    data = np.ascontiguousarray(data, dtype=np.complex128)
    h = lib.oracle_ilu(n, _ptr(indptr), _ptr(indices), _ptr(data), float(droptol),
                       1 if restrict_pattern else 0)
    try:
        ln, un, st = C.c_long(), C.c_long(), C.c_int()
        lib.oracle_ilu_sizes(h, C.byref(ln), C.byref(un), C.byref(st))
        li = np.zeros(n + 1, dtype=np.int64)
        ui = np.zeros(n + 1, dtype=np.int64)
        lj = np.empty(ln.value, dtype=np.int64)
        lv = np.empty(ln.value, dtype=np.complex128)
        uj = np.empty(un.value, dtype=np.int64)
        uv = np.empty(un.value, dtype=np.complex128)
        lib.oracle_ilu_copy(h, _ptr(li), _ptr(lj), _ptr(lv), _ptr(ui), _ptr(uj), _ptr(uv))
    finally:
        lib.oracle_ilu_free(h)
    return li, lj, lv, ui, uj, uv, st.value


def _tri(name, fac, out):
    """One of precond.py:129-173 on every column of the (n, r) C-ordered block."""
    lib = _lib()
    i, j, v = fac
    fn = getattr(lib, name)
    n, r = out.shape
    for c in range(r):
        col = out[:, c]
        fn(n, _ptr(i), _ptr(j), _ptr(v), C.c_void_p(col.ctypes.data), r)
    return out


class Factorization:
    """precond.py:183-269"""

    def __init__(self, kind, n, lu=None, chol=None, diag_inv=None, sign=1.0):
        self.kind = kind
        self.n = n
        self.lu = lu
        self.chol = chol
        self.diag_inv = diag_inv
        self.sign = sign

    @property
    def is_spd_capable(self):
        return self.kind in ("none", "jacobi", "ic0", "ict")

    @staticmethod
    def _block(x):
        squeeze = (np.ndim(x) == 1)
        out = np.array(x, dtype=np.complex128, copy=True, ndmin=2)
        if squeeze:
            out = out.reshape(-1, 1)
        return np.ascontiguousarray(out), squeeze

    def _chol_solves(self, out):
        _tri("oracle_solve_lower", self.chol, out)
        _tri("oracle_solve_lower_transposed", self.chol, out)
        return out

    def apply(self, x):
        """precond.py:224-240"""
        out, squeeze = self._block(x)
        if self.kind == "jacobi":
            out *= self.diag_inv[:, None]
        elif self.kind in ("ilu0", "ilut"):
            li, lj, lv, ui, uj, uv = self.lu
            _tri("oracle_solve_unit_lower", (li, lj, lv), out)
            _tri("oracle_solve_upper", (ui, uj, uv), out)
        elif self.kind in ("ic0", "ict"):
            self._chol_solves(out)
            if self.sign < 0:
                out = -out
        return out[:, 0] if squeeze else out

    def apply_spd(self, x):
        """precond.py:242-256"""
        if not self.is_spd_capable:
            raise ValueError(f"kind {self.kind!r} has no SPD split form")
        out, squeeze = self._block(x)
        if self.kind == "jacobi":
            out *= np.abs(self.diag_inv)[:, None]
        elif self.kind in ("ic0", "ict"):
            self._chol_solves(out)
        return out[:, 0] if squeeze else out


def chol_from_ilu(kind, n, lu, sign):
    """precond.py:279-304: G = L sqrt(D), diagonal last in every row."""
    li, lj, lv, ui, uj, uv = lu
    d = uv[ui[:-1]]
    if np.any(d.real <= 0.0) or np.any(np.abs(d.imag) > 1e-10 * np.abs(d.real)):
        raise FactorizationBreakdown("matrix is not positive definite up to dropping")
    sq = np.sqrt(d.real).astype(np.complex128)
    counts = np.diff(li)
    gi = np.zeros(n + 1, dtype=np.int64)
    gi[1:] = np.cumsum(counts + 1)
    gj = np.empty(int(gi[-1]), dtype=np.int64)
    gv = np.empty(int(gi[-1]), dtype=np.complex128)
    rows = np.repeat(np.arange(n), counts)
    pos = np.arange(li[-1]) + rows            # every earlier row holds one diagonal slot
    gj[pos] = lj
    gv[pos] = lv * sq[lj]
    dpos = gi[1:] - 1
    gj[dpos] = np.arange(n)
    gv[dpos] = sq
    return Factorization(kind, n, chol=(gi, gj, gv), sign=sign)


def assembled(op):
    """The explicit matrix of an oracle ShiftedOp: base + shift * mass on the
    merged pattern (sparse.py:138-155), conjugate-transposed on the adjoint side
    (sparse.py:183-190)."""
    base = sp.csr_matrix(op.base)
    mass = sp.eye(op.n, op.n, format="csr") if op.mass is None else sp.csr_matrix(op.mass)
    shift = complex(op.shift)
    if shift.imag == 0.0:
        mat = base + shift.real * mass
    else:
        mat = base.astype(complex) + shift * mass
    mat = sp.csr_matrix(mat)
    if op.adjoint:
        mat = sp.csr_matrix(mat.conj().T)
    mat.sort_indices()
    return mat


def factorize(matrix, kind, droptol=0.0):
    """precond.py:307-357 on a scipy CSR matrix."""
    if kind not in KINDS:
        raise ValueError(f"unknown preconditioner kind {kind!r}")
    matrix = sp.csr_matrix(matrix)
    n = matrix.shape[0]
    if matrix.shape[1] != n:
        raise ValueError("preconditioned matrix must be square")
    if kind == "none":
        return Factorization("none", n)
    if kind == "jacobi":
        d = matrix.diagonal().astype(np.complex128)
        if np.any(np.abs(d) < PIVOT_TINY):
            raise FactorizationBreakdown("zero diagonal entry for Jacobi")
        return Factorization("jacobi", n, diag_inv=1.0 / d)
    work, sign = matrix, 1.0
    if kind in ("ic0", "ict"):
        if np.real(matrix.diagonal()).sum() < 0.0:
            work, sign = sp.csr_matrix(-matrix), -1.0
    restrict = kind in ("ilu0", "ic0")
    tol = 0.0 if restrict else float(droptol)
    *lu, status = ilu_kernel(n, work.indptr, work.indices, work.data, tol, restrict)
    if status != 0:
        raise FactorizationBreakdown(f"zero pivot in {kind} factorization")
    if kind in ("ilu0", "ilut"):
        return Factorization(kind, n, lu=tuple(lu))
    return chol_from_ilu(kind, n, tuple(lu), sign)
