"""CPU ORACLE for the inexact low-rank Sylvester ADI hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module, and only as the checker or the timed CPU baseline -- never as the thing
measured or shipped.  The product package (``paper_2312_02891_b200``) does not
import it.

This is a numpy/scipy restatement of the reference package ``sylvadi``
(``/root/reference/pkg/src/sylvadi``; every function cites the file:line it
follows) plus the NEW inner solver the B200 build uses: Jacobi-right-
preconditioned GMRES(m)/FGMRES(m), batched per column, with CGS2
orthogonalisation and Givens least squares.  The reference has no GMRES
(SURVEY.md D1); the GMRES contract below is SURVEY.md section 8a "Algorithm
contract for a8" and is the one the CUDA kernels implement.

Parity pinning (see tests/test_oracle_pin.py and tests/golden/make_golden.py):
* tolerance strategies, residual norms, shifted apply, Jacobi, BiCGstab and
  the ADI driver are pinned against outputs of the reference itself, run in
  the build container, committed as fixtures under tests/golden/;
* the known-answer values of the reference's own tests (test_adi.py:47-52,
  84-88, 92-102, 29-37, 155-167; test_precond.py:105-108) are re-checked;
* the GMRES restatement has no reference counterpart -- its solutions are
  cross-checked against dense solves and against scipy.sparse.linalg.gmres,
  and at the ADI level against the reference's own BiCGstab path (same outer
  step count, residual below tau).
"""

import math
import time
import warnings

import numpy as np
import scipy.sparse as sp

# -- constants --------------------------------------------------------------

#: adi.py:27
C_BOUND = 2.0 + math.sqrt(2.0)

STRATEGIES = ("fixed", "dynamic_mid", "dynamic_mid_bl", "dynamic_b",
              "dynamic_b_bl", "exact_direct", "direct_a_iter_b",
              "iter_a_direct_b")
#: adi.py:41-46
BL_STRATEGIES = {"dynamic_mid_bl", "dynamic_b_bl", "direct_a_iter_b",
                 "iter_a_direct_b"}

#: krylov.py:79
BREAKDOWN_TINY = 1e-290
#: GMRES lucky-breakdown threshold (new code)
GMRES_LUCKY = 1e-14


# -- small dense helpers -----------------------------------------------------

def gamma(alpha, beta):
    """adi.py:49-51"""
    return -(complex(beta) + complex(alpha))


def block_norm(x):
    """adi.py:54-59: spectral norm of a thin block."""
    x = np.atleast_2d(x)
    if x.size == 0:
        return 0.0
    return float(np.linalg.svd(x, compute_uv=False)[0])


def computed_residual_norm(w, t):
    """adi.py:62-70: ||w t^*||_2 via thin QR of both factors."""
    w = np.atleast_2d(w)
    t = np.atleast_2d(t)
    if w.size == 0 or t.size == 0:
        return 0.0
    rw = np.linalg.qr(w, mode="r")
    rt = np.linalg.qr(t, mode="r")
    return float(np.linalg.svd(rw @ rt.conj().T, compute_uv=False)[0])


# -- configuration -----------------------------------------------------------

class Config:
    """adi.py:130-168 (AdiConfig defaults and validation)."""

    def __init__(self, outer_tolerance=1e-8, kmax=50, xi=1.0,
                 strategy="dynamic_mid_bl", fixed_delta=None,
                 delta_min_A=None, delta_max_A=0.1, delta_min_B=None,
                 delta_max_B=0.1, gap_budget=None, max_inner_iterations=1000):
        strategy = str(getattr(strategy, "value", strategy))
        if strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {strategy!r}")
        if not (0.0 < outer_tolerance < 1.0):
            raise ValueError("outer_tolerance must be in (0, 1)")
        if not (0.0 < xi <= 1.0):
            raise ValueError("xi must be in (0, 1]")
        if kmax < 1:
            raise ValueError("kmax must be >= 1")
        self.outer_tolerance = outer_tolerance
        self.kmax = kmax
        self.xi = xi
        self.strategy = strategy
        self.fixed_delta = outer_tolerance / 20.0 if fixed_delta is None else fixed_delta
        self.delta_min_A = outer_tolerance / 20.0 if delta_min_A is None else delta_min_A
        self.delta_min_B = outer_tolerance / 20.0 if delta_min_B is None else delta_min_B
        self.delta_max_A = delta_max_A
        self.delta_max_B = delta_max_B
        for lo, hi in ((self.delta_min_A, self.delta_max_A),
                       (self.delta_min_B, self.delta_max_B)):
            if not (0.0 < lo <= hi):
                raise ValueError("need 0 < delta_min <= delta_max")
        self.gap_budget = gap_budget
        self.max_inner_iterations = max_inner_iterations


def tolerance_budget(cfg, k, u_prev=0.0, v_prev=0.0, gap_budget=None):
    """adi.py:347-361: eps-hat^(1) (uniform) or eps-hat^(2) (back-looking)."""
    eps = cfg.gap_budget if gap_budget is None else gap_budget
    if eps is None:
        raise ValueError("gap budget is not set")
    if cfg.strategy in BL_STRATEGIES:
        return (1.0 / C_BOUND) * abs(
            cfg.xi * k * eps / (2.0 * C_BOUND * cfg.kmax) - u_prev - v_prev)
    return cfg.xi * eps / (2.0 * C_BOUND**2 * cfg.kmax)


def tolB_from_tolA(delta_A, eps_check, c_check, norm_t, norm_w):
    """adi.py:364-369"""
    val = (eps_check - c_check * delta_A * norm_t) / \
          (c_check * (2.0 * delta_A + norm_w))
    return max(val, 0.0)


def choose_tolerances(cfg, k, norm_w, norm_t, eps_hat):
    """adi.py:372-408.  Returns (delta_A, delta_B, clamped_A, clamped_B)."""
    s = cfg.strategy
    if s == "exact_direct":
        return 0.0, 0.0, False, False
    if s == "fixed":
        return cfg.fixed_delta, cfg.fixed_delta, False, False
    if s == "direct_a_iter_b":
        raw = eps_hat / max(norm_w, 1e-300)
        dB = min(max(raw, cfg.delta_min_B), cfg.delta_max_B)
        return 0.0, dB, False, raw < cfg.delta_min_B
    if s == "iter_a_direct_b":
        raw = eps_hat / max(norm_t, 1e-300)
        dA = min(max(raw, cfg.delta_min_A), cfg.delta_max_A)
        return dA, 0.0, raw < cfg.delta_min_A, False
    if s in ("dynamic_mid", "dynamic_mid_bl"):
        mid = 0.5 * (min(cfg.delta_max_A, eps_hat / max(norm_t, 1e-300))
                     - cfg.delta_min_A)
        dA = max(mid, cfg.delta_min_A)
        rawB = (eps_hat - dA * norm_t) / (2.0 * dA + norm_w)
        dB = max(min(rawB, cfg.delta_max_B), cfg.delta_min_B)
        return dA, dB, mid < cfg.delta_min_A, rawB < cfg.delta_min_B
    dB = cfg.delta_min_B
    rawA = (eps_hat - dB * norm_w) / (norm_t + 2.0 * dB)
    dA = max(min(rawA, cfg.delta_max_A), cfg.delta_min_A)
    return dA, dB, rawA < cfg.delta_min_A, False


# -- operators ---------------------------------------------------------------

class ShiftedOp:
    """sparse.py:158-206: (base + shift*mass) or its conjugate transpose.

    ``base``/``mass`` are real scipy CSR matrices (mass None = identity).
    """

    def __init__(self, base, mass, shift, adjoint=False):
        self.base = sp.csr_matrix(base)
        self.mass = None if mass is None else sp.csr_matrix(mass)
        self.shift = complex(shift)
        self.adjoint = bool(adjoint)
        self.n = self.base.shape[0]
        self._baseT = self.base.T.tocsr() if adjoint else None
        self._massT = (self.mass.T.tocsr()
                       if (adjoint and self.mass is not None) else None)

    def apply(self, x):
        """sparse.py:192-206 (transpose applied through a stored CSR of the
        transpose instead of scipy's CSC view: same products, summation in
        column-index order)."""
        x = np.asarray(x)
        if x.ndim == 1:
            x = x.reshape(-1, 1)
        if self.adjoint:
            out = (self._baseT @ x).astype(complex)
            sig = np.conj(self.shift)
            out += sig * (x if self.mass is None else self._massT @ x)
        else:
            out = (self.base @ x).astype(complex)
            out += self.shift * (x if self.mass is None else self.mass @ x)
        return out

    def diagonal(self):
        """Diagonal of the assembled operator (sparse.py:183-190,138-155),
        conjugated on the adjoint side."""
        d = self.base.diagonal().astype(complex)
        md = np.ones(self.n) if self.mass is None else self.mass.diagonal()
        d = d + self.shift * md
        return np.conj(d) if self.adjoint else d


class FactorizationBreakdown(RuntimeError):
    """precond.py FactorizationBreakdown"""


def jacobi_dinv(op):
    """precond.py:272-276: dinv = 1/diag(assembled op); breakdown if |d|<1e-300."""
    d = op.diagonal().astype(np.complex128)
    if np.any(np.abs(d) < 1e-300):
        raise FactorizationBreakdown("zero diagonal entry for Jacobi")
    return 1.0 / d


# -- inner solve results ------------------------------------------------------

class InnerResult:
    """krylov.py:41-70"""

    def __init__(self, solution, residual, iterations, tol_col):
        self.solution = solution
        self.residual = residual
        self.achieved_residual_norms = np.linalg.norm(residual, axis=0)
        self.iterations = np.asarray(iterations, dtype=np.int64)
        self.converged = self.achieved_residual_norms <= tol_col

    @property
    def total_iterations(self):
        return int(self.iterations.sum())

    @property
    def block_residual_norm(self):
        if self.residual.size == 0:
            return 0.0
        return float(np.linalg.svd(self.residual, compute_uv=False)[0])


def _finalize(op, rhs, x, iters, tol_col):
    """krylov.py:61-70"""
    res = rhs - op.apply(x)
    return InnerResult(x, res, iters, tol_col)


# -- BiCGstab (the reference's own inner solver) ------------------------------

def _bicgstab_column(op, dinv, b, tol, maxit):
    """krylov.py:82-157 -- right-preconditioned BiCGstab, one column."""
    n = b.shape[0]
    x = np.zeros(n, dtype=np.complex128)
    r = b.copy()
    if np.linalg.norm(r) <= tol:
        return x, 0
    if dinv is None:
        pre = lambda v: v.copy()                      # noqa: E731
    elif hasattr(dinv, "apply"):                      # incomplete factorisation (oracle/precond.py)
        pre = lambda v: dinv.apply(v)                 # noqa: E731
    else:
        pre = lambda v: v * dinv                      # noqa: E731
    rhat = r.copy()
    rho = alpha = omega = 1.0 + 0.0j
    v = np.zeros(n, dtype=np.complex128)
    p = np.zeros(n, dtype=np.complex128)
    it = 0
    restarted = False
    while it < maxit:
        rho_new = np.vdot(rhat, r)
        scale = np.linalg.norm(rhat) * np.linalg.norm(r)
        if abs(rho_new) <= BREAKDOWN_TINY * max(scale, 1.0):
            if restarted:
                break
            rhat = r.copy()
            rho = alpha = omega = 1.0 + 0.0j
            v[:] = 0.0
            p[:] = 0.0
            restarted = True
            continue
        beta = (rho_new / rho) * (alpha / omega)
        p = r + beta * (p - omega * v)
        phat = pre(p)
        v = op.apply(phat[:, None])[:, 0]
        denom = np.vdot(rhat, v)
        if abs(denom) <= BREAKDOWN_TINY * max(scale, 1.0):
            if restarted:
                break
            rhat = r.copy()
            rho = alpha = omega = 1.0 + 0.0j
            v[:] = 0.0
            p[:] = 0.0
            restarted = True
            continue
        alpha = rho_new / denom
        s = r - alpha * v
        x += alpha * phat
        it += 1
        if np.linalg.norm(s) <= tol:
            return x, it
        shat = pre(s)
        t = op.apply(shat[:, None])[:, 0]
        tt = np.vdot(t, t).real
        if tt <= BREAKDOWN_TINY:
            if restarted:
                break
            rhat = s.copy()
            r = s
            rho = alpha = omega = 1.0 + 0.0j
            v[:] = 0.0
            p[:] = 0.0
            restarted = True
            continue
        omega = np.vdot(t, s) / tt
        if abs(omega) <= BREAKDOWN_TINY:
            if restarted:
                break
            rhat = s.copy()
            r = s
            rho = alpha = omega = 1.0 + 0.0j
            v[:] = 0.0
            p[:] = 0.0
            restarted = True
            continue
        x += omega * shat
        r = s - omega * t
        rho = rho_new
        if np.linalg.norm(r) <= tol:
            return x, it
    return x, it


def bicgstab(op, rhs, abs_tolerance, max_iterations=1000, dinv=None):
    """krylov.py:160-184 (per-column loop with drift-resume)."""
    rhs = _check_request(op, rhs, abs_tolerance)
    r = rhs.shape[1]
    tol_col = abs_tolerance / r
    x = np.zeros_like(rhs)
    iters = np.zeros(r, dtype=np.int64)
    for c in range(r):
        xc, it = _bicgstab_column(op, dinv, rhs[:, c], tol_col, max_iterations)
        budget = max_iterations - it
        true_res = rhs[:, c] - op.apply(xc[:, None])[:, 0]
        while np.linalg.norm(true_res) > tol_col and budget > 0 and it > 0:
            dx, extra = _bicgstab_column(op, dinv, true_res, tol_col, budget)
            if extra == 0:
                break
            xc = xc + dx
            it += extra
            budget -= extra
            true_res = rhs[:, c] - op.apply(xc[:, None])[:, 0]
        x[:, c] = xc
        iters[c] = it
    return _finalize(op, rhs, x, iters, tol_col)


# -- MINRES (the reference's inner solver for Hermitian sides) -----------------

def _minres_column(op, dinv, b, tol, maxit):
    """krylov.py:187-268 -- split-preconditioned MINRES (Paige-Saunders), one
    column.  The SPD split of Jacobi is |dinv| (precond.py:242-256); dinv None
    is the identity."""
    n = b.shape[0]
    x = np.zeros(n, dtype=np.complex128)
    if np.linalg.norm(b) <= tol:
        return x, 0
    if hasattr(dinv, "apply_spd"):                    # Cholesky kinds: (G G^H)^-1 (precond.py:242-256)
        psolve = lambda v: dinv.apply_spd(v)          # noqa: E731
    else:
        pabs = None if dinv is None else np.abs(dinv)
        psolve = (lambda v: v.copy()) if pabs is None else (lambda v: v * pabs)
    r1 = b.astype(np.complex128)
    y = psolve(r1)
    beta1_sq = np.vdot(r1, y).real
    if beta1_sq <= 0.0:
        raise RuntimeError("MINRES preconditioner is not positive definite")
    beta1 = np.sqrt(beta1_sq)
    oldb, beta, dbar, epsln, phibar = 0.0, beta1, 0.0, 0.0, beta1
    cs, sn = -1.0, 0.0
    w = np.zeros(n, dtype=np.complex128)
    w2 = np.zeros(n, dtype=np.complex128)
    r2 = r1.copy()
    ratio = np.linalg.norm(b) / beta1
    check_at = tol / max(ratio, 1e-300)
    it = 0
    while it < maxit:
        it += 1
        s = 1.0 / beta
        v = s * y
        y = op.apply(v[:, None])[:, 0]
        if it >= 2:
            y -= (beta / oldb) * r1
        alfa = np.vdot(v, y).real
        y -= (alfa / beta) * r2
        r1 = r2
        r2 = y
        y = psolve(r2)
        oldb = beta
        beta = np.sqrt(max(np.vdot(r2, y).real, 0.0))
        oldeps = epsln
        delta = cs * dbar + sn * alfa
        gbar = sn * dbar - cs * alfa
        epsln = sn * beta
        dbar = -cs * beta
        gamma = max(np.hypot(gbar, beta), 1e-300)
        cs = gbar / gamma
        sn = beta / gamma
        phi = cs * phibar
        phibar = sn * phibar
        w1 = w2
        w2 = w
        w = (v - oldeps * w1 - delta * w2) / gamma
        x = x + phi * w
        if phibar <= check_at:
            nr = np.linalg.norm(b - op.apply(x[:, None])[:, 0])
            if nr <= tol:
                return x, it
            if phibar <= 1e-300:
                break
            check_at = min(check_at, 0.5 * tol * phibar / nr)
        if beta <= 1e-300:
            break
    return x, it


def minres(op, rhs, abs_tolerance, max_iterations=1000, dinv=None):
    """krylov.py:271-287 (per column, no resume)."""
    rhs = _check_request(op, rhs, abs_tolerance)
    r = rhs.shape[1]
    tol_col = abs_tolerance / r
    x = np.zeros_like(rhs)
    iters = np.zeros(r, dtype=np.int64)
    for c in range(r):
        xc, it = _minres_column(op, dinv, rhs[:, c], tol_col, max_iterations)
        x[:, c] = xc
        iters[c] = it
    return _finalize(op, rhs, x, iters, tol_col)


def is_symmetric(matrix, tol=1e-12):
    """adi.py:413-419"""
    csr = sp.csr_matrix(matrix)
    diff = (csr - csr.T).tocoo()
    if diff.nnz == 0:
        return True
    scale = max(np.abs(csr.data).max(initial=0.0), 1.0)
    return bool(np.abs(diff.data).max(initial=0.0) <= tol * scale)


def _check_request(op, rhs, abs_tolerance):
    """krylov.py:25-35 (InnerSolveRequest validation)."""
    rhs = np.asarray(rhs, dtype=np.complex128)
    if rhs.ndim == 1:
        rhs = rhs.reshape(-1, 1)
    if rhs.shape[0] != op.n:
        raise ValueError("rhs rows do not match operator size")
    if abs_tolerance <= 0.0:
        raise ValueError("abs_tolerance must be positive")
    if not np.all(np.isfinite(rhs)):
        raise ValueError("rhs contains non-finite entries")
    return rhs


# -- GMRES(m) / FGMRES(m): the new inner solver (SURVEY 8a contract) ----------

def givens(f, g):
    """Complex Givens rotation (zlartg convention): returns (c, s, r) with
    [c s; -conj(s) c] [f; g] = [r; 0], c real >= 0."""
    af, ag = abs(f), abs(g)
    if ag == 0.0:
        return 1.0, 0.0j, f
    if af == 0.0:
        return 0.0, np.conj(g) / ag, complex(ag)
    nrm = math.hypot(af, ag)
    alpha = f / af
    return af / nrm, alpha * np.conj(g) / nrm, alpha * nrm


def _gmres_column(op, dinv, b, tol, m, maxit, flexible, orth="cgs2"):
    """One column of Jacobi-right-preconditioned GMRES(m) from x0 = 0.

    Iteration = one Arnoldi step (u = D^-1 v_j, w = Op u, CGS2, Givens).
    ``orth="dcgs2"`` replaces the second Gram-Schmidt pass by its Gram-matrix
    form (the device engine's choice): with G = V^H V kept up to date one
    column late (G[:, j] = V^H v_j, formed in the same sweep as h1 = V^H w),
    h2 = h1 - G h1 equals V^H (w - V h1) in exact arithmetic, so
    w <- w - V (h1 + h2) in ONE update sweep (two basis sweeps per step
    instead of four; the delayed re-orthogonalisation of Swirydowicz et al.).
    A cycle ends when |g_{j+1}| <= tol, j+1 == m, a lucky breakdown
    (h_{j+1,j} <= GMRES_LUCKY*||w_pre||) or the iteration cap; then
    x += D^-1 V y (GMRES) / Z y (FGMRES) and the TRUE residual b - Op x is
    recomputed; the column stops once it is <= tol or the cap is reached,
    otherwise GMRES restarts from the true residual (the analogue of the
    reference's drift-resume, krylov.py:170-181).
    Returns (x, iterations, residual).
    """
    n = b.shape[0]
    x = np.zeros(n, dtype=np.complex128)
    r = b.astype(np.complex128).copy()
    beta = np.linalg.norm(r)
    it = 0
    if beta <= tol:                         # krylov.py:87-88 analogue
        return x, 0, r
    while True:
        V = np.zeros((m + 1, n), dtype=np.complex128)
        Gm = np.zeros((m + 1, m + 1), dtype=np.complex128) if orth == "dcgs2" else None
        Z = np.zeros((m, n), dtype=np.complex128) if flexible else None
        H = np.zeros((m + 1, m), dtype=np.complex128)
        cs = np.zeros(m)
        sn = np.zeros(m, dtype=np.complex128)
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(m):
            u = dinv * V[j]
            if flexible:
                Z[j] = u
            w = op.apply(u[:, None])[:, 0]
            wpre = np.linalg.norm(w)
            if orth == "dcgs2":
                gcol = V[:j + 1].conj() @ V[j]
                Gm[:j + 1, j] = gcol
                Gm[j, :j + 1] = np.conj(gcol)
                h1 = V[:j + 1].conj() @ w
                h = h1 + (h1 - Gm[:j + 1, :j + 1] @ h1)
                w = w - V[:j + 1].T @ h
            else:
                h = V[:j + 1].conj() @ w
                w = w - V[:j + 1].T @ h
                h2 = V[:j + 1].conj() @ w
                w = w - V[:j + 1].T @ h2
                h = h + h2
            hn = np.linalg.norm(w)
            col = np.zeros(m + 1, dtype=np.complex128)
            col[:j + 1] = h
            col[j + 1] = hn
            for i in range(j):
                a, bb = col[i], col[i + 1]
                col[i] = cs[i] * a + sn[i] * bb
                col[i + 1] = -np.conj(sn[i]) * a + cs[i] * bb
            c_, s_, rr = givens(col[j], col[j + 1])
            cs[j], sn[j] = c_, s_
            col[j], col[j + 1] = rr, 0.0
            H[:, j] = col
            g[j + 1] = -np.conj(s_) * g[j]
            g[j] = c_ * g[j]
            it += 1
            k = j + 1
            est = abs(g[j + 1])
            if hn > 0.0:
                V[j + 1] = w / hn
            if (est <= tol or k == m or hn <= GMRES_LUCKY * wpre
                    or it >= maxit):
                break
        y = _back_substitute(H[:k, :k], g[:k])
        if flexible:
            x = x + Z[:k].T @ y
        else:
            x = x + dinv * (V[:k].T @ y)
        r = b - op.apply(x[:, None])[:, 0]
        beta = np.linalg.norm(r)
        if beta <= tol or it >= maxit:
            return x, it, r


def _back_substitute(R, g):
    k = R.shape[0]
    y = np.zeros(k, dtype=np.complex128)
    for i in range(k - 1, -1, -1):
        acc = g[i] - R[i, i + 1:k] @ y[i + 1:k]
        y[i] = acc / R[i, i]
    return y


def gmres(op, rhs, abs_tolerance, max_iterations=1000, dinv=None,
          restart=50, flexible=False, orth="cgs2"):
    """Batched-by-column GMRES with the reference's result contract
    (krylov.py:41-70, per-column target abs_tolerance/r, krylov.py:164)."""
    rhs = _check_request(op, rhs, abs_tolerance)
    r = rhs.shape[1]
    tol_col = abs_tolerance / r
    if dinv is None:
        dinv = np.ones(op.n, dtype=np.complex128)
    x = np.zeros_like(rhs)
    iters = np.zeros(r, dtype=np.int64)
    for c in range(r):
        xc, it, _ = _gmres_column(op, dinv, rhs[:, c], tol_col, restart,
                                  max_iterations, flexible, orth)
        x[:, c] = xc
        iters[c] = it
    return _finalize(op, rhs, x, iters, tol_col)


# -- inner-solver bindings and the ADI driver ---------------------------------

class Binding:
    """adi.py:422-488 restricted to the iterative Jacobi path.

    ``solver`` is "bicgstab" (the reference's own choice for unsymmetric
    operators, adi.py:486-488), "minres", "reference" (the reference's
    dispatch: MINRES for a symmetric side at a real shift, else BiCGstab,
    adi.py:468-488) or "gmres"/"fgmres" (the B200 build's solver).
    """

    def __init__(self, side, base, mass, solver="gmres", max_iterations=1000,
                 restart=50, precond="jacobi", orth="cgs2", droptol=0.1):
        self.droptol = droptol
        self.side = side
        self.base = base
        self.mass = mass
        self.solver = solver
        self.max_iterations = max_iterations
        self.restart = restart
        self.precond = precond
        self.orth = orth
        self._ops = {}

    def _op(self, shift):
        shift = complex(shift)
        hit = self._ops.get(shift)
        if hit is None:
            op = ShiftedOp(self.base, self.mass, shift, adjoint=(self.side == "B"))
            if self.precond in ("ilu0", "ilut", "ic0", "ict"):
                # adi.py:453-466: factorise the assembled matrix, Jacobi on breakdown
                from . import precond as _pc
                try:
                    dinv = _pc.factorize(_pc.assembled(op), self.precond, self.droptol)
                except _pc.FactorizationBreakdown as exc:
                    warnings.warn(f"{self.side}-side {self.precond} factorization broke down "
                                  f"at shift {shift} ({exc}); falling back to Jacobi")
                    dinv = jacobi_dinv(op)
            else:
                dinv = jacobi_dinv(op) if self.precond == "jacobi" else None
            hit = (op, dinv)
            self._ops[shift] = hit
        return hit

    def uses_minres(self, shift):
        """adi.py:468-472 (iterative mode)."""
        if self.solver == "minres":
            return True
        return (self.solver == "reference" and complex(shift).imag == 0.0
                and self.precond in ("none", "jacobi", "ic0", "ict") and is_symmetric(self.base)
                and (self.mass is None or is_symmetric(self.mass)))

    def solve(self, shift, rhs, delta):
        op, dinv = self._op(shift)
        if self.uses_minres(shift):
            return minres(op, rhs, delta, self.max_iterations, dinv)
        if self.solver in ("bicgstab", "reference"):
            return bicgstab(op, rhs, delta, self.max_iterations, dinv)
        return gmres(op, rhs, delta, self.max_iterations, dinv,
                     restart=self.restart, flexible=(self.solver == "fgmres"),
                     orth=self.orth)


class StepRec:
    """adi.py:193-210"""
    FIELDS = ("step", "scaled_res", "delta_A", "delta_B", "achieved_rA",
              "achieved_rB", "inner_it_A", "inner_it_B", "u", "v", "wall_ms",
              "a_converged", "b_converged", "clamped_A_min", "clamped_B_min")

    def __init__(self, **kw):
        for f in self.FIELDS:
            setattr(self, f, kw[f])


class Run:
    def __init__(self):
        self.records = []
        self.converged = False
        self.outer_iterations = 0
        self.final_scaled_residual = float("nan")
        self.rhs_norm = 0.0
        self.wall_ms = 0.0
        self.Z = None
        self.Y = None
        self.gammas = []
        self.w = None
        self.t = None
        self.u = 0.0
        self.v = 0.0

    @property
    def sum_inner_A(self):
        return sum(r.inner_it_A for r in self.records)

    @property
    def sum_inner_B(self):
        return sum(r.inner_it_B for r in self.records)

    def dense(self):
        """adi.py:269-272"""
        gd = np.repeat(np.asarray(self.gammas, dtype=complex),
                       self.Z.shape[1] // max(len(self.gammas), 1))
        return (self.Z * gd[None, :]) @ self.Y.conj().T


def run_adi(A, B, f, g, cfg, pairs, bind_A, bind_B, M=None, C=None,
            cyclic=True):
    """adi.py:553-607 (run_with_state) with adi.py:510-537 (adi_step) inlined.

    ``pairs`` is the shift list (ShiftSequence.pairs, shifts.py:31-51).
    """
    t_start = time.perf_counter()
    f = np.atleast_2d(np.asarray(f))
    g = np.atleast_2d(np.asarray(g))
    r = f.shape[1]
    w = f.astype(complex)
    t = g.astype(complex)
    Zs, Ys = [], []
    out = Run()
    res0 = computed_residual_norm(f, g)
    out.rhs_norm = res0
    if res0 == 0.0:
        out.converged = True
        out.final_scaled_residual = 0.0
        out.Z = np.zeros((f.shape[0], 0), complex)
        out.Y = np.zeros((g.shape[0], 0), complex)
        return out
    gap = cfg.gap_budget if cfg.gap_budget is not None else cfg.outer_tolerance * res0
    u = v = 0.0
    res = res0
    k_done = 0
    MT = None if M is None else sp.csr_matrix(M)
    CT = None if C is None else sp.csr_matrix(C).T.tocsr()
    for k in range(1, cfg.kmax + 1):
        t0 = time.perf_counter()
        eps_hat = tolerance_budget(cfg, k, u, v, gap)
        nw, nt = block_norm(w), block_norm(t)
        dA, dB, clA, clB = choose_tolerances(cfg, k, nw, nt, eps_hat)
        i = k - 1
        if i >= len(pairs):
            if not cyclic:
                raise IndexError("shift sequence exhausted")
            i %= len(pairs)
        alpha, beta = complex(pairs[i][0]), complex(pairs[i][1])
        ra = bind_A.solve(beta, w, dA if dA > 0 else 1.0)
        rb = bind_B.solve(alpha, t, dB if dB > 0 else 1.0)
        z, y = ra.solution, rb.solution
        gam = gamma(alpha, beta)
        Mz = z if MT is None else MT @ z
        Cty = y if CT is None else CT @ y
        rA, rB = ra.block_residual_norm, rb.block_residual_norm
        w = w + gam * Mz
        t = t + np.conj(gam) * Cty
        u += abs(gam) * block_norm(Mz) * rB
        v += abs(gam) * block_norm(Cty) * rA
        Zs.append(z)
        Ys.append(y)
        out.gammas.append(gam)
        k_done = k
        res = computed_residual_norm(w, t)
        rec = StepRec(step=k, scaled_res=res / res0, delta_A=dA, delta_B=dB,
                      achieved_rA=rA, achieved_rB=rB,
                      inner_it_A=ra.total_iterations,
                      inner_it_B=rb.total_iterations, u=u, v=v,
                      wall_ms=1000.0 * (time.perf_counter() - t0),
                      a_converged=bool(np.all(ra.converged)),
                      b_converged=bool(np.all(rb.converged)),
                      clamped_A_min=clA, clamped_B_min=clB)
        out.records.append(rec)
        if not (rec.a_converged and rec.b_converged):
            warnings.warn(f"inner solver missed its target at step {k}; "
                          "continuing with the achieved residual")
        if res < cfg.outer_tolerance * res0:
            break
    out.converged = bool(res < cfg.outer_tolerance * res0)
    out.outer_iterations = k_done
    out.final_scaled_residual = res / res0
    out.wall_ms = 1000.0 * (time.perf_counter() - t_start)
    out.Z = np.hstack(Zs) if Zs else np.zeros((f.shape[0], 0), complex)
    out.Y = np.hstack(Ys) if Ys else np.zeros((g.shape[0], 0), complex)
    out.w, out.t, out.u, out.v = w, t, u, v
    return out


def factored_relative_difference(Z1, g1, Y1, Z2, g2, Y2):
    """||Z1 G1 Y1^* - Z2 G2 Y2^*||_F / ||Z2 G2 Y2^*||_F without forming X
    (the residual_gap technique, adi.py:674-679, with Frobenius norms).
    g1/g2 are the expanded Gamma diagonals."""
    L = np.hstack([Z1 * np.asarray(g1)[None, :], -Z2 * np.asarray(g2)[None, :]])
    Rr = np.hstack([Y1, Y2])
    rl = np.linalg.qr(L, mode="r")
    rr = np.linalg.qr(Rr, mode="r")
    num = np.linalg.norm(rl @ rr.conj().T)
    l2 = np.linalg.qr(Z2 * np.asarray(g2)[None, :], mode="r")
    r2 = np.linalg.qr(Y2, mode="r")
    den = np.linalg.norm(l2 @ r2.conj().T)
    return float(num / den)


def true_residual_norm(A, B, f, g, Z, Y, gdiag, M=None, C=None, tol=1e-6,
                       max_iterations=200):
    """Spectral norm of R = A X C + M X B + f g^*, X = Z diag(gdiag) Y^*, by
    power iteration on x -> R^*(R x) (adi.py:682-726: x0 = ones/sqrt(m),
    lambda = ||R x||^2, stop on a relative change <= tol).  Real coefficient
    matrices, so the adjoint products are transposes (adi.py:729-733)."""
    f = np.asarray(f, dtype=complex)
    g = np.asarray(g, dtype=complex)
    gd = np.asarray(gdiag, dtype=complex)

    def apply_R(x):
        Cx = x if C is None else C @ x
        Bx = B @ x
        out = f @ (g.conj().T @ x)
        if Z.shape[1]:
            out = out + A @ (Z @ (gd[:, None] * (Y.conj().T @ Cx)))
            zb = Z @ (gd[:, None] * (Y.conj().T @ Bx))
            out = out + (zb if M is None else M @ zb)
        return out

    def apply_Rh(x):
        out = g @ (f.conj().T @ x)
        if Z.shape[1]:
            ya = Y @ (np.conj(gd)[:, None] * (Z.conj().T @ (A.T @ x)))
            out = out + (ya if C is None else C.T @ ya)
            mx = x if M is None else M.T @ x
            out = out + B.T @ (Y @ (np.conj(gd)[:, None] * (Z.conj().T @ mx)))
        return out

    m = g.shape[0]
    x = np.ones((m, 1), dtype=complex) / np.sqrt(m)
    lam = 0.0
    for _ in range(max_iterations):
        Rx = apply_R(x)
        y = apply_Rh(Rx)
        lam_new = float(np.linalg.norm(Rx) ** 2)
        ny = np.linalg.norm(y)
        if ny == 0.0:
            return 0.0
        x = y / ny
        if lam > 0.0 and abs(lam_new - lam) <= tol * lam_new:
            lam = lam_new
            break
        lam = lam_new
    return float(np.sqrt(lam))


def residual_gap(A, B, S_A, S_B, Z, Y, gammas, r, M=None, C=None):
    """||eta^A + eta^B||_2 (adi.py:655-679): [S^A G, M Z G] [C^T Y, S^B]^* in
    factored form through thin QR of both factors and an SVD of the small
    core.  S_A / S_B: the retained inner residual blocks (n x kr / m x kr)."""
    if len(gammas) == 0:
        return 0.0
    gd = np.repeat(np.asarray(gammas, dtype=complex), r)
    MZ = Z if M is None else M @ Z
    CtY = Y if C is None else C.T @ Y
    left = np.hstack([S_A * gd[None, :], MZ * gd[None, :]])
    right = np.hstack([CtY, S_B])
    rl = np.linalg.qr(left, mode="r")
    rr = np.linalg.qr(right, mode="r")
    return float(np.linalg.svd(rl @ rr.conj().T, compute_uv=False)[0])


def _sigma_matrix(shift_history, gammas, r, side):
    """sigma_alpha_matrix / sigma_beta_matrix (adi.py:612-629): the lower
    staircase, diagonal alpha_l (B side conj(beta_l)), row l left of the
    diagonal -gamma_l (B side -conj(gamma_l)), Kronecker with I_r."""
    k = len(gammas)
    base = np.zeros((k, k), dtype=complex)
    for l in range(k):
        if side == "A":
            base[l, l] = shift_history[l][0]
            base[l, :l] = -gammas[l]
        else:
            base[l, l] = np.conj(shift_history[l][1])
            base[l, :l] = -np.conj(gammas[l])
    return np.kron(base, np.eye(r))


def verify_factor_identity(A, B, S_A, S_B, Z, Y, w, t, gammas, shift_history, r,
                           M=None, C=None):
    """Normalised defect of A Z = M Z sigma_alpha + w E^T - S^A and its B-side
    analogue (adi.py:632-652), each divided by ||A||_F ||Z||_F (resp. B, Y);
    returns the larger."""
    k = len(gammas)
    if k == 0:
        return 0.0
    sa = _sigma_matrix(shift_history, gammas, r, "A")
    sb = _sigma_matrix(shift_history, gammas, r, "B")
    MZ = Z if M is None else M @ Z
    CtY = Y if C is None else C.T @ Y
    defect_a = A @ Z - MZ @ sa - np.tile(w, (1, k)) + S_A
    defect_b = B.T @ Y - CtY @ sb - np.tile(t, (1, k)) + S_B
    a_scale = np.linalg.norm(sp.csr_matrix(A).data) * max(np.linalg.norm(Z), 1e-300)
    b_scale = np.linalg.norm(sp.csr_matrix(B).data) * max(np.linalg.norm(Y), 1e-300)
    return max(np.linalg.norm(defect_a) / a_scale, np.linalg.norm(defect_b) / b_scale)


def steps_csv(run):
    """adi.py:211-239 row format without wall_ms."""
    rows = ["step,scaled_res,delta_A,delta_B,achieved_rA,achieved_rB,"
            "inner_it_A,inner_it_B,u,v"]
    for rec in run.records:
        rows.append(f"{rec.step},{rec.scaled_res:.16e},{rec.delta_A:.16e},"
                    f"{rec.delta_B:.16e},{rec.achieved_rA:.16e},"
                    f"{rec.achieved_rB:.16e},{rec.inner_it_A},{rec.inner_it_B},"
                    f"{rec.u:.16e},{rec.v:.16e}")
    return "\n".join(rows) + "\n"
