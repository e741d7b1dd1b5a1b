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


def _blocks(x, rows, r, device):
    """A factor given as device blocks, a host array or a list of host blocks ->
    list of (rows, r) complex128 device blocks."""
    import torch
    dev = torch.device("cuda", device)
    if isinstance(x, (list, tuple)):
        out = []
        for b in x:
            t = b if isinstance(b, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(np.asarray(b, dtype=complex)))
            out.append(t.to(dev).to(torch.complex128).contiguous())
        return out
    arr = np.asarray(x, dtype=complex)
    k = arr.shape[1] // r if arr.ndim == 2 and r else 0
    return [torch.from_numpy(np.ascontiguousarray(arr[:, j * r:(j + 1) * r])).to(dev)
            for j in range(k)]


def _state_factors(problem, state, device):
    """(Z blocks, Y blocks, S_A blocks, S_B blocks, w, t) on the device."""
    import torch
    r = problem.r
    zb = getattr(state, "z_blocks", None)
    yb = getattr(state, "y_blocks", None)
    Z = _blocks(zb if zb is not None else state.Z, problem.n, r, device)
    Y = _blocks(yb if yb is not None else state.Y, problem.m, r, device)
    if not state.keep_inner_residuals:
        raise ValueError("inner residual blocks were not retained")
    SA = _blocks(list(state.inner_residuals_A), problem.n, r, device)
    SB = _blocks(list(state.inner_residuals_B), problem.m, r, device)
    dev = torch.device("cuda", device)

    def vec(v):
        t = v if isinstance(v, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.asarray(v, dtype=complex)))
        return t.to(dev).to(torch.complex128).contiguous()
    return Z, Y, SA, SB, vec(state.w), vec(state.t)


def _fro2(x, device):
    return float(np.trace(gram(x, device=device)).real)


def verify_factor_identity(problem, state, device=0):
    """Normalised defect of the factor identities (adi.py:632-652)

        A Z = M Z sigma_alpha + w E^T - S^A,   B^T Y = C^T Y sigma_beta + t E^T - S^B

    on the device, block column by block column: with sigma_alpha's staircase
    (diagonal alpha_j, row l > j entry -gamma_l) block j of the A-side defect
    is  A z_j - alpha_j M z_j + sum_{l>j} gamma_l M z_l - w + S^A_j,  the
    suffix sum carried backwards in one n x r accumulator; every product and
    update is a library kernel (sad_csr_apply, sad_axpy), every norm a Gram
    (sad_gram).  Each side's defect is divided by ||A||_F ||Z||_F (resp.
    ||B||_F ||Y||_F); returns the larger, as the reference.
    """
    import torch
    from .device import axpy
    k = int(state.k)
    if k == 0:
        return 0.0
    torch.cuda.set_device(device)
    Z, Y, SA, SB, w, t = _state_factors(problem, state, device)
    hist = [(complex(a), complex(b)) for a, b in state.shift_history]
    gam = [complex(x) for x in state.gammas]

    def side(base, mass, blocks, S, last, diag, coef):
        tot = 0.0
        acc = torch.zeros_like(last)
        for j in range(k - 1, -1, -1):
            xj = blocks[j]
            mx = xj if mass is None else mass.apply(xj, transpose=base.transposed)
            d = base.apply(xj, transpose=base.transposed)
            axpy(-diag[j], mx, d, device=device)
            axpy(1.0, acc, d, device=device)
            axpy(-1.0, last, d, device=device)
            axpy(1.0, S[j], d, device=device)
            tot += _fro2(d, device)
            axpy(coef[j], mx, acc, device=device)
        return np.sqrt(tot)

    class _Side:
        def __init__(self, mat, transposed):
            self.m = None if mat is None else DeviceMatrix(mat, transpose=True, device=device)
            self.transposed = transposed

        def apply(self, x, transpose=False):
            return self.m.apply(x, transpose=transpose)

    Ad, Bd = _Side(problem.A, False), _Side(problem.B, True)
    Md = None if problem.M is None else _Side(problem.M, False)
    Cd = None if problem.C is None else _Side(problem.C, True)
    da = side(Ad, Md, Z, SA, w, [a for a, _ in hist], gam)
    db = side(Bd, Cd, Y, SB, t, [np.conj(b) for _, b in hist], [np.conj(x) for x in gam])
    za = np.sqrt(sum(_fro2(z, device) for z in Z))
    yb = np.sqrt(sum(_fro2(y, device) for y in Y))

    def fro_vals(m):
        from .device import as_csr
        return float(np.linalg.norm(as_csr(m).data))
    a_scale = fro_vals(problem.A) * max(za, 1e-300)
    b_scale = fro_vals(problem.B) * max(yb, 1e-300)
    return max(da / a_scale, db / b_scale)


def _block_gram(blocks, device, chunk_bytes=1 << 31):
    """X^H X for X = [blocks...] (rows x K, never stored): row chunks of the
    blocks concatenated and multiplied by cuBLAS ZGEMM (a plain library GEMM),
    summed over the chunks in order."""
    import torch
    rows = blocks[0].shape[0]
    K = sum(b.shape[1] for b in blocks)
    step = max(1, int(chunk_bytes // max(K * 16, 1)))
    G = torch.zeros((K, K), dtype=torch.complex128, device=blocks[0].device)
    for r0 in range(0, rows, step):
        X = torch.cat([b[r0:r0 + step] for b in blocks], dim=1)
        G += X.conj().T @ X
    return G.cpu().numpy()


def _lmax_product(Gl, Gr):
    """lambda_max(Gl Gr) for Hermitian PSD Gl, Gr, in column-scaled form:
    with Gl = Dl Gl~ Dl, Gr = Dr Gr~ Dr (unit diagonals) it is lambda_max of
    the PSD matrix  Lr^H D Gl~ D Lr  (D = Dl Dr, Gr~ = Lr Lr^H), so the wide
    range of the factors' column norms (large M Z / C^T Y columns, small
    inner-residual columns) costs no relative accuracy."""
    dl = np.sqrt(np.maximum(np.diag(Gl).real, 0.0))
    dr = np.sqrt(np.maximum(np.diag(Gr).real, 0.0))
    il = np.where(dl > 0, 1.0 / np.where(dl > 0, dl, 1.0), 0.0)
    ir = np.where(dr > 0, 1.0 / np.where(dr > 0, dr, 1.0), 0.0)
    Glt = Gl * il[:, None] * il[None, :]
    Grt = Gr * ir[:, None] * ir[None, :]
    ev, U = np.linalg.eigh(0.5 * (Grt + Grt.conj().T))
    Lr = U * np.sqrt(np.maximum(ev, 0.0))[None, :]
    D = dl * dr
    H = Lr.conj().T @ (D[:, None] * Glt * D[None, :]) @ Lr
    return float(np.max(np.linalg.eigvalsh(0.5 * (H + H.conj().T))))


def residual_gap(problem, state, device=0):
    """||eta^A + eta^B||_2 from the retained inner residual blocks
    (adi.py:655-679):  [S^A G, M Z G] [C^T Y, S^B]^*.  The reference takes a
    thin QR of each factor and an SVD of the small core; here the two Grams of
    the factors are formed on the device (row-chunked ZGEMM, so nothing n x 2kr
    is stored) and the spectral norm is sqrt(lambda_max(Gl Gr)) in
    column-scaled form (_lmax_product)."""
    import torch
    k = int(state.k)
    if k == 0:
        return 0.0
    torch.cuda.set_device(device)
    r = problem.r
    Z, Y, SA, SB, _, _ = _state_factors(problem, state, device)
    M = None if problem.M is None else DeviceMatrix(problem.M, transpose=True, device=device)
    C = None if problem.C is None else DeviceMatrix(problem.C, transpose=True, device=device)
    MZ = Z if M is None else [M.apply(z) for z in Z]
    CtY = Y if C is None else [C.apply(y, transpose=True) for y in Y]
    Gl = _block_gram(list(SA) + list(MZ), Z[0].device)
    Gr = _block_gram(list(CtY) + list(SB), Y[0].device)
    gd = np.repeat(np.asarray(state.gammas, dtype=complex), r)
    gg = np.concatenate([gd, gd])
    Gl = np.conj(gg)[:, None] * Gl * gg[None, :]     # Gram of [S^A G, M Z G]
    return float(np.sqrt(max(_lmax_product(Gl, Gr), 0.0)))


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
