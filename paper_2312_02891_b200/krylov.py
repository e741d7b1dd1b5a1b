"""The inner-solver plug-in: Jacobi-right-preconditioned GMRES/FGMRES on B200.

``GpuGmresBinding`` is a drop-in for the reference's ``SolverBinding``
(``/root/reference/pkg/src/sylvadi/adi.py:422-488``): same constructor shape
(side, base, mass, mode, precond_kind, droptol, max_iterations), the same
shift-keyed operator cache, and ``solve(shift, rhs, delta)`` returning an
``InnerSolveResult`` with the reference's fields and semantics
(``krylov.py:41-70``): true unpreconditioned residual recomputed after
termination, per-column norms, per-column iteration counts (int64) and
``converged = norm <= delta / r``.  It can be passed to the reference's own
``sylvadi.run(..., bindings=SolverBindings(A=..., B=...))`` unchanged.

The Krylov method itself is new (the reference has BiCGstab/MINRES only,
SURVEY.md D1); its contract is SURVEY.md section 8a and its CPU restatement is
``oracle/sylvadi_oracle.py:_gmres_column``.
"""

import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import (BicgWorkspace, DeviceMatrix, MinresWorkspace, DeviceOperator, GmresWorkspace, gram,
                     sigma_max_from_gram)

MAX_BLOCK = 8   # columns per device solve; wider blocks are split (columns are independent)


class _WorkspacePool:
    """Krylov workspaces are reused across bindings with the same shape
    (device, n, r, dtype, restart, flexible, engine, SM cap): a caching
    allocator for the (m+1)-block basis, like cuBLAS handles.  A workspace is
    owned by at most one binding at a time."""

    def __init__(self, keep=4):
        self.free = {}
        self.keep = keep

    def take(self, key):
        lst = self.free.get(key)
        if lst:
            return lst.pop()
        dev, n, r, dtype, restart, flexible, engine, max_sms = key
        ws = GmresWorkspace(n, r, dtype, restart, flexible, dev, engine=engine, max_sms=max_sms)
        ws.pool_key = key
        return ws

    def give(self, ws):
        key = getattr(ws, "pool_key", None)
        if key is None:
            return
        lst = self.free.setdefault(key, [])
        if len(lst) < self.keep:
            lst.append(ws)

    def clear(self):
        self.free = {}


_POOL = _WorkspacePool()


@dataclass
class InnerSolveResult:
    """Mirror of krylov.py:41-58."""
    solution: np.ndarray
    residual: np.ndarray
    achieved_residual_norms: np.ndarray
    iterations: np.ndarray
    converged: np.ndarray

    @property
    def total_iterations(self):
        return int(self.iterations.sum())

    @property
    def block_residual_norm(self):
        if self.residual.size == 0:
            return 0.0
        return float(np.linalg.svd(self.residual, compute_uv=False)[0])


@dataclass
class DeviceSolveResult:
    """Device-resident variant: solution/residual stay torch tensors."""
    solution: object
    residual: object
    achieved_residual_norms: np.ndarray
    iterations: np.ndarray
    converged: np.ndarray
    residual_gram: np.ndarray = None

    @property
    def total_iterations(self):
        return int(self.iterations.sum())

    @property
    def block_residual_norm(self):
        if self.residual_gram is None:
            self.residual_gram = gram(self.residual)
        return sigma_max_from_gram(self.residual_gram)


def validate_request(n, rhs, abs_tolerance):
    """InnerSolveRequest.__post_init__ (krylov.py:25-35)."""
    rhs = np.asarray(rhs, dtype=np.complex128)
    if rhs.ndim == 1:
        rhs = rhs.reshape(-1, 1)
    if rhs.shape[0] != n:
        raise ValueError("rhs rows do not match operator size")
    if abs_tolerance <= 0.0:
        raise ValueError("abs_tolerance must be positive")
    if not np.all(np.isfinite(rhs)):
        raise ValueError("rhs contains non-finite entries")
    return rhs


PHASE_A = {"auto": -1, "tma": 0, "direct": 1}


SOLVERS = ("gmres", "bicgstab", "minres", "reference")
#: precond.py:15 kinds that carry triangular factors
FACTOR_KINDS = ("ilu0", "ilut", "ic0", "ict")


def _side_symmetric(mat, tol=1e-12):
    """adi.py:413-419 on a host matrix (DeviceMatrix: its recorded flag)."""
    if isinstance(mat, DeviceMatrix):
        return bool(getattr(mat, "symmetric", False))
    import scipy.sparse as sp
    csr = sp.csr_matrix(mat.scipy() if hasattr(mat, "scipy") else mat)
    diff = (csr - csr.T).tocoo()
    if diff.nnz == 0:
        return True
    scale = max(np.abs(csr.data).max(initial=0.0), 1.0)
    return bool(np.abs(diff.data).max(initial=0.0) <= tol * scale)


class GpuGmresBinding:
    """Per-side GPU inner solver with shift-keyed operator cache (adi.py:422-488).

    Extra keyword-only knobs (no slot in the reference's AdiConfig):
    ``restart`` (GMRES restart length m) and ``flexible`` (FGMRES form);
    engine tuning: ``engine``, ``max_sms`` and ``phase_a`` (persistent engine's
    basis sweep: "tma" ring, "direct" loads for small slabs, or "auto").
    """

    def __init__(self, side, base, mass, mode="iterative", precond_kind="jacobi",
                 droptol=0.1, max_iterations=1000, *, restart=50, flexible=False,
                 device=0, engine="persistent", max_sms=0, phase_a="auto", solver="gmres"):
        if side not in ("A", "B"):
            raise ValueError("side must be 'A' or 'B'")
        if mode != "iterative":
            raise NotImplementedError(
                "direct (sparse LU) inner solves are outside the GPU hot path; "
                "use the reference's SolverBinding for exact_direct")
        if precond_kind not in _lib.PRECOND_CODES:
            raise ValueError(f"unknown preconditioner kind {precond_kind!r}")
        if solver not in SOLVERS:
            raise ValueError(f"solver must be one of {SOLVERS}")
        if precond_kind in FACTOR_KINDS and solver == "gmres":
            raise ValueError("incomplete-factorisation preconditioners (the reference's "
                             "ilu0/ilut/ic0/ict) run with the reference's solvers: "
                             "solver='reference', 'bicgstab' or 'minres'")
        self.solver = solver
        self.side = side
        self.mode = mode
        self.precond_kind = precond_kind
        self.droptol = droptol
        self.max_iterations = int(max_iterations)
        self.restart = int(restart)
        self.flexible = bool(flexible)
        self.device = device
        self.engine = engine
        self.max_sms = int(max_sms)
        if phase_a not in PHASE_A:
            raise ValueError(f"phase_a must be one of {sorted(PHASE_A)}")
        self.phase_a = phase_a
        adjoint = (side == "B")
        # solver="reference": the reference's own dispatch (adi.py:468-488),
        # MINRES for a symmetric side at a real shift, BiCGstab otherwise
        self.symmetric = False
        if solver == "reference":
            self.symmetric = _side_symmetric(base) and (mass is None or _side_symmetric(mass))
        self.base = base if isinstance(base, DeviceMatrix) else DeviceMatrix(base, adjoint, device)
        self.mass = (None if mass is None else
                     mass if isinstance(mass, DeviceMatrix) else DeviceMatrix(mass, adjoint, device))
        self.n = self.base.shape[0]
        self._operators = {}
        self._workspaces = {}

    # -- caches -------------------------------------------------------------
    def operator(self, shift):
        shift = complex(shift)
        op = self._operators.get(shift)
        if op is None:
            adj = (self.side == "B")
            try:
                op = DeviceOperator(self.base, self.mass, shift, adjoint=adj,
                                    precond_kind=self.precond_kind, droptol=self.droptol)
            except _lib.FactorizationBreakdown as exc:
                if self.precond_kind in FACTOR_KINDS:
                    # adi.py:458-465: fall back to Jacobi (its own breakdown propagates)
                    warnings.warn(f"{self.side}-side {self.precond_kind} factorization broke "
                                  f"down at shift {shift} ({exc}); falling back to Jacobi")
                    op = DeviceOperator(self.base, self.mass, shift, adjoint=adj,
                                        precond_kind="jacobi")
                elif self.precond_kind == "none":
                    raise
                else:
                    warnings.warn(f"{self.side}-side jacobi factorization broke down at shift "
                                  f"{shift}; continuing without preconditioner")
                    op = DeviceOperator(self.base, self.mass, shift, adjoint=adj,
                                        precond_kind="none")
            self._operators[shift] = op
        return op

    def uses_minres(self, shift):
        """adi.py:468-472 (mode is always "iterative" here)."""
        if self.solver == "minres":
            return True
        return (self.solver == "reference" and self.symmetric
                and complex(shift).imag == 0.0
                and self.precond_kind in ("none", "jacobi", "ic0", "ict"))

    def kind_for(self, shift):
        """The inner algorithm a solve at ``shift`` runs."""
        if self.solver in ("gmres", "bicgstab", "minres"):
            return self.solver
        return "minres" if self.uses_minres(shift) else "bicgstab"

    def workspace(self, r, dtype, kind=None):
        kind = self.solver if kind is None else kind
        key = (kind, r, dtype)
        ws = self._workspaces.get(key)
        if ws is None:
            if kind == "bicgstab":
                ws = BicgWorkspace(self.n, r, dtype, self.device)
            elif kind == "minres":
                ws = MinresWorkspace(self.n, r, dtype, self.device)
            else:
                ws = _POOL.take((self.device, self.n, r, dtype, self.restart, self.flexible,
                                 self.engine, self.max_sms))
            self._workspaces[key] = ws
        ws.set_option(_lib.SAD_OPT_DIRECT_A, PHASE_A[self.phase_a])
        return ws

    def release(self):
        """Return the Krylov workspaces to the shared pool now (the next
        binding of the same shape reuses them without a device allocation)."""
        for ws in getattr(self, "_workspaces", {}).values():
            if isinstance(ws, GmresWorkspace):
                _POOL.give(ws)
        self._workspaces = {}

    def __del__(self):
        self.release()

    # -- solves -------------------------------------------------------------
    def solve_device(self, shift, rhs, delta, x=None, res=None, stream=None,
                     fixed_steps=None):
        """Solve with device blocks (torch, (n, r) float64/complex128).

        ``delta`` is the block target; the per-column target is delta / r
        (krylov.py:164).  Returns a DeviceSolveResult.
        """
        import torch
        if delta <= 0.0:
            raise ValueError("abs_tolerance must be positive")
        n, r = rhs.shape
        if n != self.n:
            raise ValueError("rhs rows do not match operator size")
        op = self.operator(shift)
        if rhs.dtype == torch.float64 and not op.is_real:
            raise ValueError("complex shift requires a complex128 block")
        dtype = _lib.SAD_F64 if rhs.dtype == torch.float64 else _lib.SAD_C128
        x = torch.empty_like(rhs) if x is None else x
        res = torch.empty_like(rhs) if res is None else res
        tol_col = float(delta) / r
        iters = np.zeros(r, dtype=np.int64)
        norms = np.zeros(r, dtype=np.float64)
        conv = np.zeros(r, dtype=bool)
        for c0 in range(0, r, MAX_BLOCK):
            c1 = min(r, c0 + MAX_BLOCK)
            width = c1 - c0
            if width == r:
                b_, x_, res_ = rhs, x, res
            else:
                b_ = rhs[:, c0:c1].contiguous()
                x_ = torch.empty_like(b_)
                res_ = torch.empty_like(b_)
            ws = self.workspace(width, dtype, self.kind_for(shift))
            if fixed_steps is not None and self.solver != "gmres":
                raise ValueError("fixed_steps applies to GMRES only")
            if fixed_steps is None:
                it, nr, cv = ws.solve(op, b_, x_, res_, tol_col, self.max_iterations, stream)
            else:
                nr, _ = ws.fixed(op, b_, x_, res_, fixed_steps, stream)
                it = np.full(width, fixed_steps, dtype=np.int64)
                cv = nr <= tol_col
            if width != r:
                x[:, c0:c1] = x_
                res[:, c0:c1] = res_
            iters[c0:c1], norms[c0:c1], conv[c0:c1] = it, nr, cv
        return DeviceSolveResult(solution=x, residual=res, achieved_residual_norms=norms,
                                 iterations=iters, converged=conv)

    def begin_device(self, shift, rhs, delta, x, res, stream=None):
        """Enqueue a device solve (r <= 8 columns); pair with ``end_device``."""
        import torch
        if delta <= 0.0:
            raise ValueError("abs_tolerance must be positive")
        n, r = rhs.shape
        if n != self.n or r > MAX_BLOCK:
            raise ValueError("begin_device needs an (n, r<=8) block")
        if self.solver != "gmres" or self.engine != "persistent":
            raise ValueError("begin_device/end_device need the persistent GMRES engine")
        op = self.operator(shift)
        if rhs.dtype == torch.float64 and not op.is_real:
            raise ValueError("complex shift requires a complex128 block")
        dtype = _lib.SAD_F64 if rhs.dtype == torch.float64 else _lib.SAD_C128
        ws = self.workspace(r, dtype)
        ws.launch(op, rhs, x, float(delta) / r, self.max_iterations, stream)
        return (ws, x, res, stream)

    def end_device(self, token):
        ws, x, res, stream = token
        it, nr, cv = ws.finish(res, stream)
        return DeviceSolveResult(solution=x, residual=res, achieved_residual_norms=nr,
                                 iterations=it, converged=cv)

    def solve(self, shift, rhs, delta):
        """SolverBinding.solve (adi.py:473-488) on host numpy blocks."""
        import torch
        rhs = validate_request(self.n, rhs, delta)
        op = self.operator(shift)
        real = op.is_real and not np.any(rhs.imag)
        dev = torch.device("cuda", self.device)
        b = torch.from_numpy(np.ascontiguousarray(rhs.real if real else rhs)).to(dev)
        out = self.solve_device(shift, b, delta)
        torch.cuda.current_stream(dev).synchronize()
        sol = out.solution.cpu().numpy().astype(np.complex128)
        res = out.residual.cpu().numpy().astype(np.complex128)
        tol_col = delta / rhs.shape[1]
        norms = np.linalg.norm(res, axis=0)
        return InnerSolveResult(solution=sol, residual=res, achieved_residual_norms=norms,
                                iterations=out.iterations, converged=norms <= tol_col)


@dataclass
class SolverBindings:
    """adi.py:491-494"""
    A: object
    B: object


def make_gpu_bindings(problem, config, restart=50, flexible=False, device=0,
                      engine="persistent", solver="gmres"):
    """GPU counterpart of make_bindings (adi.py:497-505)."""
    kind_a = getattr(config, "precond_kind_A", "jacobi")
    kind_b = getattr(config, "precond_kind_B", "jacobi")
    tol_a = getattr(config, "precond_droptol_A", 0.1)
    tol_b = getattr(config, "precond_droptol_B", 0.1)
    maxit = getattr(config, "max_inner_iterations", 1000)
    return SolverBindings(
        A=GpuGmresBinding("A", problem.A, problem.M, "iterative", kind_a, tol_a,
                          max_iterations=maxit, restart=restart, flexible=flexible,
                          device=device, engine=engine, solver=solver),
        B=GpuGmresBinding("B", problem.B, problem.C, "iterative", kind_b, tol_b,
                          max_iterations=maxit, restart=restart, flexible=flexible,
                          device=device, engine=engine, solver=solver))
