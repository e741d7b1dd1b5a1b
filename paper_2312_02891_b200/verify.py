"""Device-side verification of a low-rank ADI solution.

``true_residual_norm`` is the reference's diagnostic (adi.py:682-726) with the
same signature, meaning and stopping rule: the spectral norm of the true
Sylvester residual

    R = A Z G Y^* C + M Z G Y^* B + f g^*        (G = diag(gamma_k I_r))

by power iteration on x -> R^*(R x), the residual matrix never formed.  Here
every product runs on the device: the sparse products through the library's
CSR kernels (spmv / spmv_transpose, sparse.py:118-135), the factor products
``Y^* v`` / ``Z c`` through ``sad_ts_hgemv`` / ``sad_ts_gemv``, and the norms
through ``sad_gram``; the host only keeps the K-vectors and the scalars.  At
configs 3-5 this is the size-independent correctness check of a converged
run (the reference's CPU power iteration streams the n x kr factors up to 400
times per call).
"""

import ctypes

import numpy as np

from . import _lib
from .device import DeviceMatrix, gram


class _Factor:
    """A low-rank factor (rows x K) as one contiguous device matrix."""

    def __init__(self, blocks_or_array, rows, device):
        import torch
        dev = torch.device("cuda", device)
        if isinstance(blocks_or_array, (list, tuple)):
            blocks = [b.to(dev) for b in blocks_or_array]
            t = torch.cat(blocks, dim=1) if blocks else torch.zeros((rows, 0), device=dev)
        else:
            arr = np.asarray(blocks_or_array)
            if not np.iscomplexobj(arr):
                arr = arr.astype(np.float64)
            t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        if t.dtype not in (torch.float64, torch.complex128):
            t = t.to(torch.complex128)
        self.t = t.contiguous()
        self.rows, self.K = self.t.shape
        self.dtype = _lib.SAD_F64 if self.t.dtype == torch.float64 else _lib.SAD_C128

    def hgemv(self, ctx, V, stream):
        """X^H V (K x nvec, host complex128) for an (rows, nvec) complex block."""
        nvec = V.shape[1]
        out = np.empty((self.K, nvec), dtype=np.complex128)
        _lib.check(_lib.load().sad_ts_hgemv(ctx, self.rows, self.K, self.K, self.dtype,
                                            ctypes.c_void_p(self.t.data_ptr()), nvec,
                                            ctypes.c_void_p(V.data_ptr()), out.ctypes.data,
                                            stream), ctx)
        return out

    def gemv(self, ctx, C, Y, stream, accumulate=False):
        """Y (+)= X C for host coefficients C (K x nvec)."""
        C = np.ascontiguousarray(C, dtype=np.complex128)
        _lib.check(_lib.load().sad_ts_gemv(ctx, self.rows, self.K, self.K, self.dtype,
                                           ctypes.c_void_p(self.t.data_ptr()), C.shape[1],
                                           C.ctypes.data, ctypes.c_void_p(Y.data_ptr()),
                                           1 if accumulate else 0, stream), ctx)
        return Y


def _mat(m, device):
    return None if m is None else DeviceMatrix(m, transpose=True, device=device)


def true_residual_norm(problem, solution, tol=1e-6, max_iterations=200, device=0):
    """Spectral norm of A X C + M X B + f g^*, X = Z G Y^*, by power iteration
    (adi.py:682-726: start x = ones/sqrt(m), lambda = ||R x||^2, stop when the
    relative change is <= tol or after max_iterations; returns sqrt(lambda)).

    ``problem``: SylvesterProblem (host scipy matrices); ``solution``: a
    LowRankSolution with device blocks (from ``run``/``DeviceAdi``) or host
    factors.
    """
    import torch
    from .device import current_stream_handle
    ctx = _lib.context(device)
    torch.cuda.set_device(device)
    stream = current_stream_handle()
    n, m, r = problem.n, problem.m, problem.r
    A, B = _mat(problem.A, device), _mat(problem.B, device)
    M, C = _mat(problem.M, device), _mat(problem.C, device)
    dev = torch.device("cuda", device)
    f = _Factor(np.asarray(problem.f, dtype=complex), n, device)
    g = _Factor(np.asarray(problem.g, dtype=complex), m, device)
    zb, yb = getattr(solution, "device_blocks", (None, None))
    if zb is not None and yb is not None:
        Z, Y = _Factor(list(zb), n, device), _Factor(list(yb), m, device)
    else:
        Z, Y = _Factor(solution.Z, n, device), _Factor(solution.Y, m, device)
    gd = solution.gamma_diag()
    K = Z.K
    c128 = torch.complex128

    def norm2(v):
        return float(gram(v, device=device).real[0, 0])

    def apply_R(x):
        Cx = x if C is None else C.apply(x)
        Bx = x if B is None else B.apply(x)
        out = torch.empty((n, 1), dtype=c128, device=dev)
        f.gemv(ctx, g.hgemv(ctx, x, stream), out, stream)          # f (g^* x)
        if K:
            both = torch.cat([Cx, Bx], dim=1).contiguous()
            yc = Y.hgemv(ctx, both, stream) * gd[:, None]            # G (Y^* [Cx, Bx])
            zz = torch.empty((n, 2), dtype=c128, device=dev)
            Z.gemv(ctx, yc, zz, stream)                              # Z G Y^* [Cx, Bx]
            zc = zz[:, 0:1].contiguous()
            zb_ = zz[:, 1:2].contiguous()
            out += A.apply(zc)
            out += zb_ if M is None else M.apply(zb_)
        return out

    def apply_Rh(x):
        out = torch.empty((m, 1), dtype=c128, device=dev)
        g.gemv(ctx, f.hgemv(ctx, x, stream), out, stream)           # g (f^* x)
        if K:
            Ahx = A.apply(x, transpose=True)                          # real matrices: A^* = A^T
            Mhx = x if M is None else M.apply(x, transpose=True)
            both = torch.cat([Ahx, Mhx], dim=1).contiguous()
            za = Z.hgemv(ctx, both, stream) * np.conj(gd)[:, None]   # conj(G) Z^* [A^*x, M^*x]
            yy = torch.empty((m, 2), dtype=c128, device=dev)
            Y.gemv(ctx, za, yy, stream)
            ya = yy[:, 0:1].contiguous()
            ym = yy[:, 1:2].contiguous()
            out += ya if C is None else C.apply(ya, transpose=True)
            out += B.apply(ym, transpose=True)
        return out

    x = torch.full((m, 1), 1.0 / np.sqrt(m), dtype=c128, device=dev)
    lam = 0.0
    for _ in range(max_iterations):
        Rx = apply_R(x)
        y = apply_Rh(Rx)
        lam_new = norm2(Rx)
        ny = np.sqrt(norm2(y))
        if ny == 0.0:
            return 0.0
        x = y / ny
        if lam > 0.0 and abs(lam_new - lam) <= tol * lam_new:
            lam = lam_new
            break
        lam = lam_new
    return float(np.sqrt(lam))
