"""Device objects: CSR matrices, shifted operators, Krylov workspaces, blocks.

Thin RAII wrappers over the C-ABI handles.  Device memory for vector blocks
is torch tensors (plumbing only); the arithmetic runs in libsylvadi_b200.so.
"""

import ctypes
import math

import numpy as np
import scipy.sparse as sp

from . import _lib

_KIND = {"none": _lib.SAD_PRECOND_NONE, "jacobi": _lib.SAD_PRECOND_JACOBI}


def as_csr(mat):
    """scipy CSR (canonical) from a scipy matrix, a reference SparseMatrix
    (anything with ``.scipy()``) or a dense array."""
    if hasattr(mat, "scipy"):
        mat = mat.scipy()
    if sp.issparse(mat):
        csr = sp.csr_matrix(mat)
    else:
        arr = np.asarray(mat)
        if arr.ndim != 2:
            raise ValueError("expected a 2-d matrix")
        csr = sp.csr_matrix(arr)
    if not (csr.has_sorted_indices and csr.has_canonical_format):
        csr = csr.copy()
        csr.sum_duplicates()
        csr.sort_indices()
    if np.iscomplexobj(csr.data):
        raise ValueError("coefficient matrices must be real (sparse.py:33-35)")
    return csr


def torch_dtype(dtype):
    import torch
    return torch.float64 if dtype == _lib.SAD_F64 else torch.complex128


def current_stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class DeviceMatrix:
    """Real CSR matrix resident on the device (optionally with its transpose)."""

    def __init__(self, mat, transpose=False, device=0):
        csr = as_csr(mat)
        self.shape = csr.shape
        self.nnz = int(csr.nnz)
        self.device = device
        self.has_transpose = bool(transpose)
        self._ctx = _lib.context(device)
        lib = _lib.load()
        rp = np.ascontiguousarray(csr.indptr, dtype=np.int32)
        ci = np.ascontiguousarray(csr.indices, dtype=np.int32)
        va = np.ascontiguousarray(csr.data, dtype=np.float64)
        h = ctypes.c_void_p()
        rc = lib.sad_csr_create(self._ctx, csr.shape[0], csr.shape[1], self.nnz,
                                rp.ctypes.data, ci.ctypes.data, va.ctypes.data,
                                1 if transpose else 0, ctypes.byref(h))
        _lib.check(rc, self._ctx)
        self.handle = h
        self.diagonal = csr.diagonal()

    @property
    def nrows(self):
        return self.shape[0]

    def apply(self, x, y=None, transpose=False, stream=None):
        """y = A x (or A^T x) for an (n, r) torch block."""
        import torch
        dtype = _lib.SAD_F64 if x.dtype == torch.float64 else _lib.SAD_C128
        rows = self.shape[1] if transpose else self.shape[0]
        if y is None:
            y = torch.empty((rows, x.shape[1]), dtype=x.dtype, device=x.device)
        rc = _lib.load().sad_csr_apply(self.handle, 1 if transpose else 0, x.shape[1], dtype,
                                       x.data_ptr(), y.data_ptr(),
                                       current_stream_handle(stream))
        _lib.check(rc, self._ctx)
        return y

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.load().sad_csr_destroy(h)
            except Exception:
                pass
            self.handle = None


class DevicePrecond:
    """Incomplete factorisation of ``base + shift*mass`` (or its conjugate
    transpose): ``factorize(op.assembled(), kind, droptol)`` (precond.py:307-357)
    with the factors on the device (sad_pc_create).  Raises
    FactorizationBreakdown like the reference."""

    def __init__(self, base, mass, shift, adjoint, kind, droptol):
        if kind not in ("ilu0", "ilut", "ic0", "ict"):
            raise ValueError(f"{kind!r} is not an incomplete factorisation kind")
        self.kind, self.droptol = kind, float(droptol)
        self.n = base.shape[0]
        self._ctx = base._ctx
        shift = complex(shift)
        h = ctypes.c_void_p()
        rc = _lib.load().sad_pc_create(self._ctx, base.handle,
                                       None if mass is None else mass.handle, shift.real,
                                       shift.imag, 1 if adjoint else 0,
                                       _lib.PRECOND_CODES[kind], self.droptol, ctypes.byref(h))
        _lib.check(rc, self._ctx)
        self.handle = h
        info = np.zeros(8, dtype=np.int64)
        _lib.check(_lib.load().sad_pc_info(h, info.ctypes.data), self._ctx)
        self.nnz = (int(info[2]), int(info[3]))
        self.is_complex = bool(info[4])
        self.levels = (int(info[5]), int(info[6]))
        self.sign = float(info[7])

    @property
    def is_spd_capable(self):
        return self.kind in ("ic0", "ict")

    def factor(self, which=0):
        """The reference's raw triplets (indptr, indices, data complex128): 0 = L
        (unit diagonal not stored) or G (diagonal last per row), 1 = U (diagonal
        first) -- IncompleteFactorization._lu / _chol (precond.py:193-202)."""
        nnz = self.nnz[which]
        ip = np.zeros(self.n + 1, dtype=np.int64)
        ix = np.zeros(max(nnz, 1), dtype=np.int64)
        dv = np.zeros(max(nnz, 1), dtype=np.complex128)
        _lib.check(_lib.load().sad_pc_get_factor(self.handle, which, ip.ctypes.data,
                                                 ix.ctypes.data, dv.ctypes.data), self._ctx)
        return ip, ix[:nnz], dv[:nnz]

    def apply(self, x, y=None, spd=False, stream=None):
        """y = M^-1 x (precond.py:224-240), or (G G^H)^-1 x with ``spd``
        (precond.py:242-256) on a device block; y may be x."""
        import torch
        dtype = _lib.SAD_F64 if x.dtype == torch.float64 else _lib.SAD_C128
        if y is None:
            y = torch.empty_like(x)
        rc = _lib.load().sad_pc_apply(self.handle, x.shape[1], dtype, x.data_ptr(), y.data_ptr(),
                                      1 if spd else 0, current_stream_handle(stream))
        _lib.check(rc, self._ctx)
        return y

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.load().sad_pc_destroy(h)
            except Exception:
                pass
            self.handle = None


class DeviceOperator:
    """``base + shift*mass`` (or its conjugate transpose) with its preconditioner
    (ShiftedOperator, sparse.py:158-206 + precond.py): none / Jacobi folded into
    the operator (device dinv), the incomplete factorisations as ``self.pc``."""

    def __init__(self, base, mass, shift, adjoint=False, precond_kind="jacobi", droptol=0.1):
        if precond_kind not in _lib.PRECOND_CODES:
            raise ValueError(f"unknown preconditioner kind {precond_kind!r}")
        self.base, self.mass = base, mass
        self.shift = complex(shift)
        self.adjoint = bool(adjoint)
        self.n = base.shape[0]
        self._ctx = base._ctx
        self.precond_kind = precond_kind
        self.pc = None
        if precond_kind not in _KIND:
            # may raise FactorizationBreakdown (the binding falls back to Jacobi)
            self.pc = DevicePrecond(base, mass, shift, adjoint, precond_kind, droptol)
        h = ctypes.c_void_p()
        rc = _lib.load().sad_op_create(self._ctx, base.handle,
                                       None if mass is None else mass.handle,
                                       self.shift.real, self.shift.imag,
                                       1 if adjoint else 0,
                                       _KIND.get(precond_kind, _lib.SAD_PRECOND_NONE),
                                       ctypes.byref(h))
        _lib.check(rc, self._ctx)
        self.handle = h
        self.is_real = (self.shift.imag == 0.0)

    def band_info(self, plan_class=0):
        """The banded SpMM plan of this operator (sad_op_band_info; built on first
        use): dict with tiles, padded entries, nnz, max local x rows, padded row
        length and rows per tile, or None when the operator runs the CSR kernels.
        plan_class 0: the stand-alone SpMM; 1: the persistent kernel's sub-phase."""
        info = np.zeros(7, dtype=np.int64)
        _lib.check(_lib.load().sad_op_band_info(self.handle, int(plan_class), info.ctypes.data),
                   self._ctx)
        if not info[0]:
            return None
        return dict(tiles=int(info[1]), entries=int(info[2]), nnz=int(info[3]),
                    xcap=int(info[4]), wmax=int(info[5]), rows=int(info[6]))

    def dinv(self):
        out = np.empty(self.n, dtype=np.complex128)
        _lib.check(_lib.load().sad_op_get_dinv(self.handle, out.ctypes.data), self._ctx)
        return out

    def apply(self, x, y=None, stream=None):
        import torch
        dtype = _lib.SAD_F64 if x.dtype == torch.float64 else _lib.SAD_C128
        if y is None:
            y = torch.empty_like(x)
        rc = _lib.load().sad_op_apply(self.handle, x.shape[1], dtype, x.data_ptr(),
                                      y.data_ptr(), current_stream_handle(stream))
        _lib.check(rc, self._ctx)
        return y

    def apply_host(self, x, out=None, stream=None):
        """y = Op x for HOST numpy blocks (n, r) float64/complex128, through
        sad_op_apply_host: chunked uploads, SpMM and downloads overlapped (pinned
        buffers, e.g. from torch's pin_memory, give full PCIe overlap)."""
        x = np.asarray(x)
        if x.ndim == 1:
            x = x.reshape(-1, 1)
        if x.dtype not in (np.float64, np.complex128) or not x.flags.c_contiguous:
            raise ValueError("x must be a C-contiguous float64 or complex128 block")
        if x.shape[0] != self.n:
            raise ValueError(f"block has {x.shape[0]} rows, operator expects {self.n}")
        if out is None:
            out = np.empty_like(x)
        if out.shape != x.shape or out.dtype != x.dtype or not out.flags.c_contiguous:
            raise ValueError("out must match x (shape, dtype, C order)")
        dtype = _lib.SAD_F64 if x.dtype == np.float64 else _lib.SAD_C128
        rc = _lib.load().sad_op_apply_host(self.handle, x.shape[1], dtype, x.ctypes.data,
                                           out.ctypes.data, current_stream_handle(stream))
        _lib.check(rc, self._ctx)
        return out

    def residual(self, b, x, y=None, stream=None):
        import torch
        dtype = _lib.SAD_F64 if x.dtype == torch.float64 else _lib.SAD_C128
        if y is None:
            y = torch.empty_like(x)
        rc = _lib.load().sad_op_residual(self.handle, x.shape[1], dtype, b.data_ptr(),
                                         x.data_ptr(), y.data_ptr(),
                                         current_stream_handle(stream))
        _lib.check(rc, self._ctx)
        return y

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.load().sad_op_destroy(h)
            except Exception:
                pass
            self.handle = None


ENGINES = {"multi": _lib.SAD_ENGINE_MULTI, "persistent": _lib.SAD_ENGINE_PERSISTENT}


def _no_pc(op):
    if getattr(op, "pc", None) is not None:
        raise ValueError("incomplete-factorisation preconditioners run with the reference's "
                         "solvers (solver='bicgstab', 'minres' or 'reference'), not with GMRES")


class GmresWorkspace:
    """(restart+1) basis blocks (+ restart Z blocks for FGMRES) on the device.

    engine "persistent" (default): the whole solve is one cooperative kernel
    with delayed-Gram CGS2 (two basis sweeps per step); "multi": one launch per
    phase with classical CGS2 (four sweeps), host-polled between cycles.
    ``max_sms`` caps the SMs a persistent solve occupies (0 = all)."""

    def __init__(self, n, r, dtype, restart, flexible, device=0, engine="persistent",
                 max_sms=0):
        self.n, self.r, self.dtype = n, r, dtype
        self.restart, self.flexible = restart, bool(flexible)
        self._ctx = _lib.context(device)
        h = ctypes.c_void_p()
        rc = _lib.load().sad_gmres_create(self._ctx, n, r, dtype, restart,
                                          1 if flexible else 0, ctypes.byref(h))
        _lib.check(rc, self._ctx)
        self.handle = h
        self.set_option(_lib.SAD_OPT_ENGINE, ENGINES[engine])
        self.engine = engine
        if max_sms:
            self.set_option(_lib.SAD_OPT_MAX_SMS, int(max_sms))

    def set_option(self, key, value):
        _lib.check(_lib.load().sad_gmres_set_option(self.handle, int(key), int(value)),
                   self._ctx)

    def profile(self, enable):
        """Enable/disable profiling; returns the 13 counters accumulated so far."""
        out = np.zeros(13, dtype=np.float64)
        _lib.check(_lib.load().sad_gmres_profile(self.handle, 1 if enable else 0,
                                                 out.ctypes.data), self._ctx)
        return out

    @property
    def nbytes(self):
        return int(_lib.load().sad_gmres_bytes(self.handle))

    def solve(self, op, rhs, x, res, tol_col, maxit, stream=None):
        """Returns (iterations int64[r], residual norms float64[r], converged bool[r])."""
        _no_pc(op)
        r = self.r
        iters = np.zeros(r, dtype=np.int64)
        norms = np.zeros(r, dtype=np.float64)
        conv = np.zeros(r, dtype=np.uint8)
        rc = _lib.load().sad_gmres_solve(
            self.handle, op.handle, rhs.data_ptr(), x.data_ptr(),
            None if res is None else res.data_ptr(), float(tol_col), int(maxit),
            current_stream_handle(stream), iters.ctypes.data, norms.ctypes.data,
            conv.ctypes.data)
        _lib.check(rc, self._ctx)
        return iters, norms, conv.astype(bool)

    def launch(self, op, rhs, x, tol_col, maxit, stream=None):
        """Enqueue a solve (returns immediately for the persistent engine)."""
        _no_pc(op)
        rc = _lib.load().sad_gmres_launch(self.handle, op.handle, rhs.data_ptr(), x.data_ptr(),
                                          float(tol_col), int(maxit),
                                          current_stream_handle(stream))
        _lib.check(rc, self._ctx)

    def finish(self, res, stream=None):
        """Wait for the launched solve; (iterations, residual norms, converged)."""
        r = self.r
        iters = np.zeros(r, dtype=np.int64)
        norms = np.zeros(r, dtype=np.float64)
        conv = np.zeros(r, dtype=np.uint8)
        rc = _lib.load().sad_gmres_finish(self.handle, None if res is None else res.data_ptr(),
                                          current_stream_handle(stream), iters.ctypes.data,
                                          norms.ctypes.data, conv.ctypes.data)
        _lib.check(rc, self._ctx)
        return iters, norms, conv.astype(bool)

    def fixed(self, op, rhs, x, res, steps, stream=None, timed=False):
        _no_pc(op)
        norms = np.zeros(self.r, dtype=np.float64)
        timing = np.zeros(8, dtype=np.float64)
        rc = _lib.load().sad_gmres_fixed(
            self.handle, op.handle, rhs.data_ptr(), x.data_ptr(),
            None if res is None else res.data_ptr(), int(steps),
            current_stream_handle(stream), norms.ctypes.data,
            timing.ctypes.data if timed else None)
        _lib.check(rc, self._ctx)
        return norms, timing

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.load().sad_gmres_destroy(h)
            except Exception:
                pass
            self.handle = None


class BicgWorkspace:
    """Device BiCGstab (the reference's own inner solver, krylov.py:82-184) on
    n x r blocks: seven n x r work blocks plus per-column scalars."""

    def __init__(self, n, r, dtype, device=0):
        self.n, self.r, self.dtype = n, r, dtype
        self._ctx = _lib.context(device)
        h = ctypes.c_void_p()
        _lib.check(_lib.load().sad_bicg_create(self._ctx, n, r, dtype, ctypes.byref(h)),
                   self._ctx)
        self.handle = h

    def set_option(self, key, value):
        """GMRES engine options do not apply."""

    @property
    def nbytes(self):
        return int(_lib.load().sad_bicg_bytes(self.handle))

    def solve(self, op, rhs, x, res, tol_col, maxit, stream=None):
        """Returns (iterations int64[r], residual norms float64[r], converged bool[r])."""
        r = self.r
        iters = np.zeros(r, dtype=np.int64)
        norms = np.zeros(r, dtype=np.float64)
        conv = np.zeros(r, dtype=np.uint8)
        rc = _lib.load().sad_bicg_solve_pc(
            self.handle, op.handle, None if op.pc is None else op.pc.handle,
            rhs.data_ptr(), x.data_ptr(),
            None if res is None else res.data_ptr(), float(tol_col), int(maxit),
            current_stream_handle(stream), iters.ctypes.data, norms.ctypes.data,
            conv.ctypes.data)
        _lib.check(rc, self._ctx)
        return iters, norms, conv.astype(bool)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.load().sad_bicg_destroy(h)
            except Exception:
                pass
            self.handle = None


class MinresWorkspace:
    """Device MINRES (the reference's inner solver for Hermitian sides,
    krylov.py:187-287) on n x r blocks: seven n x r work blocks plus per-column
    scalars.  Real shifts only (adi.py:468-472)."""

    def __init__(self, n, r, dtype, device=0):
        self.n, self.r, self.dtype = n, r, dtype
        self._ctx = _lib.context(device)
        h = ctypes.c_void_p()
        _lib.check(_lib.load().sad_minres_create(self._ctx, n, r, dtype, ctypes.byref(h)),
                   self._ctx)
        self.handle = h

    def set_option(self, key, value):
        """GMRES engine options do not apply."""

    @property
    def nbytes(self):
        return int(_lib.load().sad_minres_bytes(self.handle))

    def solve(self, op, rhs, x, res, tol_col, maxit, stream=None):
        """Returns (iterations int64[r], residual norms float64[r], converged bool[r])."""
        r = self.r
        iters = np.zeros(r, dtype=np.int64)
        norms = np.zeros(r, dtype=np.float64)
        conv = np.zeros(r, dtype=np.uint8)
        rc = _lib.load().sad_minres_solve_pc(
            self.handle, op.handle, None if op.pc is None else op.pc.handle,
            rhs.data_ptr(), x.data_ptr(),
            None if res is None else res.data_ptr(), float(tol_col), int(maxit),
            current_stream_handle(stream), iters.ctypes.data, norms.ctypes.data,
            conv.ctypes.data)
        _lib.check(rc, self._ctx)
        return iters, norms, conv.astype(bool)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.load().sad_minres_destroy(h)
            except Exception:
                pass
            self.handle = None


def gram(x, y=None, device=0, stream=None):
    """X^H Y (r x r complex numpy) of two device blocks."""
    import torch
    y = x if y is None else y
    r = x.shape[1]
    dtype = _lib.SAD_F64 if x.dtype == torch.float64 else _lib.SAD_C128
    out = np.zeros(r * r, dtype=np.complex128)
    ctx = _lib.context(device)
    rc = _lib.load().sad_gram(ctx, x.shape[0], r, dtype, x.data_ptr(), y.data_ptr(),
                              out.ctypes.data, current_stream_handle(stream))
    _lib.check(rc, ctx)
    return out.reshape(r, r)


def axpy(a, x, y, device=0, stream=None):
    """y += a x for device blocks (complex a only for complex blocks)."""
    import torch
    a = complex(a)
    dtype = _lib.SAD_F64 if x.dtype == torch.float64 else _lib.SAD_C128
    ctx = _lib.context(device)
    rc = _lib.load().sad_axpy(ctx, x.shape[0], x.shape[1], dtype, a.real, a.imag,
                              x.data_ptr(), y.data_ptr(), current_stream_handle(stream))
    _lib.check(rc, ctx)
    return y


def _lmax_herm2(a, b, d):
    """Largest eigenvalue of the Hermitian 2 x 2 [[a, b], [conj(b), d]] (a, d real):
    (a + d)/2 + sqrt(((a - d)/2)^2 + |b|^2) -- no cancellation for the maximum."""
    h = 0.5 * (a - d)
    return 0.5 * (a + d) + math.sqrt(h * h + (b.real * b.real + b.imag * b.imag))


def sigma_max_from_gram(G):
    """Largest singular value of a block from its Gram matrix X^H X (closed
    forms for r <= 2, the per-step host cost of the small configs)."""
    if G.size == 0:
        return 0.0
    r = G.shape[0]
    if r == 1:
        return math.sqrt(max(G[0, 0].real, 0.0))
    if r == 2:
        b = 0.5 * (complex(G[0, 1]) + complex(G[1, 0]).conjugate())
        return math.sqrt(max(_lmax_herm2(G[0, 0].real, b, G[1, 1].real), 0.0))
    ev = np.linalg.eigvalsh(0.5 * (G + G.conj().T))
    return float(np.sqrt(max(ev[-1], 0.0)))


def product_norm_from_grams(Gw, Gt):
    """||w t^*||_2 from Gw = w^H w and Gt = t^H t: sqrt(lambda_max(Gw^1/2 Gt Gw^1/2))
    (= sqrt(lambda_max(Gw Gt)); closed forms for r <= 2)."""
    r = Gw.shape[0]
    if r == 1:
        return math.sqrt(max(Gw[0, 0].real * Gt[0, 0].real, 0.0))
    if r == 2:
        # eigenvalues of Gw Gt (similar to the Hermitian PSD Gw^1/2 Gt Gw^1/2):
        # tr/2 + sqrt(tr^2/4 - det), det = det(Gw) det(Gt) >= 0
        bw = 0.5 * (complex(Gw[0, 1]) + complex(Gw[1, 0]).conjugate())
        bt = 0.5 * (complex(Gt[0, 1]) + complex(Gt[1, 0]).conjugate())
        aw, dw, at, dt = Gw[0, 0].real, Gw[1, 1].real, Gt[0, 0].real, Gt[1, 1].real
        tr = aw * at + dw * dt + 2.0 * (bw * bt.conjugate()).real
        det = max(aw * dw - abs(bw) ** 2, 0.0) * max(at * dt - abs(bt) ** 2, 0.0)
        lam = 0.5 * tr + math.sqrt(max(0.25 * tr * tr - det, 0.0))
        return math.sqrt(max(lam, 0.0))
    Gw = 0.5 * (Gw + Gw.conj().T)
    Gt = 0.5 * (Gt + Gt.conj().T)
    lam, Q = np.linalg.eigh(Gw)
    half = (Q * np.sqrt(np.clip(lam, 0.0, None))[None, :]) @ Q.conj().T
    K = half @ Gt @ half
    ev = np.linalg.eigvalsh(0.5 * (K + K.conj().T))
    return float(np.sqrt(max(ev[-1], 0.0)))


def adi_epilogue(gam, mz, res_a, w, cty, res_b, t, device=0, stream=None):
    """Fused ADI step epilogue: w += gam Mz, t += conj(gam) C^T y (in place) and
    the Gram matrices [resA, resB, Mz, C^T y, w, t] (6 x r x r complex numpy)."""
    import torch
    gam = complex(gam)
    r = w.shape[1]
    dtype = _lib.SAD_F64 if w.dtype == torch.float64 else _lib.SAD_C128
    out = np.zeros(6 * r * r, dtype=np.complex128)
    ctx = _lib.context(device)
    rc = _lib.load().sad_adi_epilogue(ctx, w.shape[0], t.shape[0], r, dtype, gam.real, gam.imag,
                                      mz.data_ptr(), res_a.data_ptr(), w.data_ptr(),
                                      cty.data_ptr(), res_b.data_ptr(), t.data_ptr(),
                                      out.ctypes.data, current_stream_handle(stream))
    _lib.check(rc, ctx)
    return out.reshape(6, r, r)
