"""Inexact low-rank ADI driver with dynamic inner tolerances, device resident.

Mirrors the reference API (``/root/reference/pkg/src/sylvadi/adi.py``) so a
caller can switch packages: ``SylvesterProblem``, ``AdiConfig``, ``Strategy``,
``ToleranceDecision``, ``StepRecord``/``SolveReport`` (same CSV schema),
``LowRankSolution``, ``AdiState``, the tolerance strategies and
``run``/``run_with_state`` with the same signature and return types.

Two execution paths:

* ``bindings=None`` (default): the DEVICE-RESIDENT driver.  w, t, the factor
  blocks z_k, y_k, the inner solves (GpuGmresBinding.solve_device, A and B
  sides concurrently on two CUDA streams), the w/t updates (adi.py:525-526)
  and every norm (r x r Gram matrices reduced on device, adi.py:54-70) stay on
  the GPU; the host only runs the scalar tolerance logic (adi.py:347-408,
  kept as in the reference) on O(r^2) numbers per outer step.
* ``bindings=...``: the host loop of the reference (adi.py:510-607) calling
  ``bindings.A.solve`` / ``bindings.B.solve`` on numpy blocks -- works with
  ``GpuGmresBinding`` or any SolverBinding-compatible object.
"""

import math
import threading
import time
import warnings
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .device import (DeviceMatrix, adi_epilogue, as_csr, axpy, gram,
                     product_norm_from_grams, sigma_max_from_gram)
from . import _lib
from .krylov import GpuGmresBinding, SolverBindings
from .shifts import ShiftSequence

#: adi.py:27 -- bound on the per-step Cayley constants
C_BOUND = 2.0 + math.sqrt(2.0)


class Strategy(str, Enum):
    """adi.py:30-38"""
    FIXED = "fixed"
    DYNAMIC_MID = "dynamic_mid"
    DYNAMIC_MID_BL = "dynamic_mid_bl"
    DYNAMIC_B = "dynamic_b"
    DYNAMIC_B_BL = "dynamic_b_bl"
    EXACT_DIRECT = "exact_direct"
    DIRECT_A_ITER_B = "direct_a_iter_b"
    ITER_A_DIRECT_B = "iter_a_direct_b"


_BACK_LOOKING = frozenset({Strategy.DYNAMIC_MID_BL, Strategy.DYNAMIC_B_BL,
                           Strategy.DIRECT_A_ITER_B, Strategy.ITER_A_DIRECT_B})


def _strategy(s):
    return Strategy(getattr(s, "value", s))


def gamma(alpha, beta):
    """Step coefficient -(alpha + beta) (adi.py:49-51)."""
    return -(complex(beta) + complex(alpha))


def block_norm(x):
    """Spectral norm of a thin host block (adi.py:54-59)."""
    x = np.atleast_2d(x)
    if x.size == 0:
        return 0.0
    return float(np.linalg.svd(x, compute_uv=False)[0])


def computed_residual_norm(w, t):
    """||w t^*||_2 of host blocks via thin QR (adi.py:62-70)."""
    w = np.atleast_2d(w)
    t = np.atleast_2d(t)
    if w.size == 0 or t.size == 0:
        return 0.0
    rw = np.linalg.qr(w, mode="r")
    rt = np.linalg.qr(t, mode="r")
    return float(np.linalg.svd(rw @ rt.conj().T, compute_uv=False)[0])


# -- problem / configuration ----------------------------------------------------

@dataclass
class SylvesterProblem:
    """``A X C + M X B = -f g^T`` (adi.py:75-127).  Matrices may be scipy
    sparse, dense arrays or the reference's SparseMatrix; M/C None = identity."""

    A: object
    B: object
    f: np.ndarray
    g: np.ndarray
    M: object = None
    C: object = None

    def __post_init__(self):
        self.A = as_csr(self.A)
        self.B = as_csr(self.B)
        self.M = None if self.M is None else as_csr(self.M)
        self.C = None if self.C is None else as_csr(self.C)
        self.f = _as_factor(self.f, self.A.shape[0])
        self.g = _as_factor(self.g, self.B.shape[0])
        if self.A.shape[0] != self.A.shape[1] or self.B.shape[0] != self.B.shape[1]:
            raise ValueError("A and B must be square")
        if self.M is not None and self.M.shape != self.A.shape:
            raise ValueError("M must match A")
        if self.C is not None and self.C.shape != self.B.shape:
            raise ValueError("C must match B")
        if self.f.shape[0] != self.A.shape[0] or self.g.shape[0] != self.B.shape[0]:
            raise ValueError("RHS factor dimensions do not match A, B")
        if self.f.shape[1] != self.g.shape[1]:
            raise ValueError("f and g must have the same number of columns")
        for name, blk in (("f", self.f), ("g", self.g)):
            if blk.shape[1] > 0 and np.any(blk != 0):
                if np.linalg.matrix_rank(blk) < blk.shape[1]:
                    raise ValueError(f"{name} is column rank deficient")

    @classmethod
    def from_reference(cls, problem):
        """Adopt a reference ``sylvadi.SylvesterProblem`` unchanged."""
        return cls(A=problem.A, B=problem.B, f=problem.f, g=problem.g,
                   M=problem.M, C=problem.C)

    @property
    def n(self):
        return self.A.shape[0]

    @property
    def m(self):
        return self.B.shape[0]

    @property
    def r(self):
        return self.f.shape[1]

    def rhs_norm(self):
        return computed_residual_norm(self.f, self.g)


def _as_factor(blk, nrows):
    blk = np.asarray(blk)
    if not np.iscomplexobj(blk):
        blk = blk.astype(float)
    blk = np.atleast_2d(blk)
    if blk.shape[0] == 1 and nrows > 1:
        blk = blk.T
    return blk


@dataclass
class AdiConfig:
    """adi.py:130-180 (same fields, defaults and validation)."""
    outer_tolerance: float = 1e-8
    kmax: int = 50
    xi: float = 1.0
    strategy: Strategy = Strategy.DYNAMIC_MID_BL
    fixed_delta: float = None
    delta_min_A: float = None
    delta_max_A: float = 0.1
    delta_min_B: float = None
    delta_max_B: float = 0.1
    gap_budget: float = None
    max_inner_iterations: int = 1000
    keep_inner_residuals: bool = False
    precond_kind_A: str = "none"
    precond_droptol_A: float = 0.1
    precond_kind_B: str = "none"
    precond_droptol_B: float = 0.1
    a_mode: str = None
    b_mode: str = None

    def __post_init__(self):
        self.strategy = _strategy(self.strategy)
        if not 0.0 < self.outer_tolerance < 1.0:
            raise ValueError("outer_tolerance must be in (0, 1)")
        if not 0.0 < self.xi <= 1.0:
            raise ValueError("xi must be in (0, 1]")
        if self.kmax < 1:
            raise ValueError("kmax must be >= 1")
        floor = self.outer_tolerance / 20.0
        if self.fixed_delta is None:
            self.fixed_delta = floor
        if self.delta_min_A is None:
            self.delta_min_A = floor
        if self.delta_min_B is None:
            self.delta_min_B = floor
        if not (0.0 < self.delta_min_A <= self.delta_max_A and
                0.0 < self.delta_min_B <= self.delta_max_B):
            raise ValueError("need 0 < delta_min <= delta_max")

    def side_mode(self, side):
        override = self.a_mode if side == "A" else self.b_mode
        if override is not None:
            return override
        s = self.strategy
        if s is Strategy.EXACT_DIRECT:
            return "direct"
        if (s is Strategy.DIRECT_A_ITER_B and side == "A") or \
           (s is Strategy.ITER_A_DIRECT_B and side == "B"):
            return "direct"
        return "iterative"


@dataclass
class ToleranceDecision:
    delta_A: float
    delta_B: float
    budget: float
    strategy: Strategy
    clamped_A_min: bool = False
    clamped_B_min: bool = False


@dataclass
class StepRecord:
    step: int
    scaled_res: float
    delta_A: float
    delta_B: float
    achieved_rA: float
    achieved_rB: float
    inner_it_A: int
    inner_it_B: int
    u: float
    v: float
    wall_ms: float
    a_converged: bool = True
    b_converged: bool = True
    clamped_A_min: bool = False
    clamped_B_min: bool = False


#: adi.py:212-213 -- the report CSV schema (unchanged)
CSV_HEADER = ("step,scaled_res,delta_A,delta_B,achieved_rA,achieved_rB,"
              "inner_it_A,inner_it_B,u,v,wall_ms")


@dataclass
class SolveReport:
    records: list = field(default_factory=list)
    converged: bool = False
    outer_iterations: int = 0
    final_scaled_residual: float = float("nan")
    rhs_norm: float = 0.0
    wall_ms: float = 0.0
    strategy: Strategy = Strategy.EXACT_DIRECT
    device_timing: dict = field(default_factory=dict)

    @property
    def sum_inner_A(self):
        return sum(r.inner_it_A for r in self.records)

    @property
    def sum_inner_B(self):
        return sum(r.inner_it_B for r in self.records)

    def to_rows(self):
        for r in self.records:
            yield (f"{r.step},{r.scaled_res:.16e},{r.delta_A:.16e},{r.delta_B:.16e},"
                   f"{r.achieved_rA:.16e},{r.achieved_rB:.16e},{r.inner_it_A},"
                   f"{r.inner_it_B},{r.u:.16e},{r.v:.16e},{r.wall_ms:.3f}")

    def to_csv(self, path):
        with open(path, "w") as fh:
            fh.write(CSV_HEADER + "\n")
            for row in self.to_rows():
                fh.write(row + "\n")


class LowRankSolution:
    """X ~= Z diag(gamma_k I_r) Y^* (adi.py:248-272).  Factors may stay on the
    device (``device_blocks``); ``Z``/``Y`` materialise host arrays lazily."""

    #: factors up to this size are concatenated on the device and downloaded in
    #: one copy; larger ones in chunks of this size
    CONCAT_BYTES = 256 << 20

    def __init__(self, Z=None, gammas=(), Y=None, r=1, z_blocks=None, y_blocks=None,
                 n=None, m=None):
        self._Z, self._Y = Z, Y
        self._zb, self._yb = z_blocks, y_blocks
        self.gammas = np.asarray(gammas, dtype=complex)
        self.r = r
        self._n, self._m = n, m

    @staticmethod
    def _stack(blocks, rows, r):
        """(rows, k*r) complex128 host array; each device block is copied
        straight into its column slice of one pinned buffer."""
        if not blocks:
            return np.zeros((rows, 0), dtype=complex)
        import torch
        k = len(blocks)
        total = rows * k * r * 16
        if total <= LowRankSolution.CONCAT_BYTES:
            dev = torch.cat(blocks, dim=1)            # (rows, k*r) contiguous on the device
            if dev.dtype != torch.complex128:
                dev = dev.to(torch.complex128)
            host = torch.empty((rows, k * r), dtype=torch.complex128, pin_memory=True)
            host.copy_(dev, non_blocking=True)        # one contiguous D2H copy
            torch.cuda.synchronize(dev.device)
            return host.numpy()
        # large factors (configs 3-5): row chunks packed on the device into the
        # host layout, double-buffered asynchronous copies into pinned staging
        # (the next chunk is packed and copied while host threads move the
        # previous one into the result, whose pages they also first-touch)
        return LowRankSolution._stack_chunked(blocks, rows, r)

    #: bytes per pinned staging buffer of the chunked download
    STAGE_BYTES = 256 << 20
    #: host threads moving staged chunks into the result array
    COPY_THREADS = 8
    _STAGING = None

    @staticmethod
    def _stack_chunked(blocks, rows, r):
        import torch
        from concurrent.futures import ThreadPoolExecutor
        k = len(blocks)
        width = k * r
        out = np.empty((rows, width), dtype=np.complex128)
        dev = blocks[0].device
        chunk = max(1, min(rows, LowRankSolution.STAGE_BYTES // (width * 16)))
        # the two pinned buffers are kept for the next download (Z, then Y)
        cache = LowRankSolution._STAGING
        if cache is None or cache[0].numel() < chunk * width:
            cache = [torch.empty(chunk * width, dtype=torch.complex128, pin_memory=True)
                     for _ in range(2)]
            LowRankSolution._STAGING = cache
        stages = [c[:chunk * width].view(chunk, width) for c in cache]
        events = [torch.cuda.Event(), torch.cuda.Event()]
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        nthr = LowRankSolution.COPY_THREADS

        def enqueue(i, r0):
            r1 = min(rows, r0 + chunk)
            with torch.cuda.stream(side):
                packed = torch.cat([b[r0:r1] for b in blocks], dim=1)
                if packed.dtype != torch.complex128:
                    packed = packed.to(torch.complex128)
                stages[i][:r1 - r0].copy_(packed, non_blocking=True)
                events[i].record(side)
            return r1

        def move(dst, src):
            np.copyto(dst, src)

        starts = list(range(0, rows, chunk))
        with ThreadPoolExecutor(max_workers=nthr) as pool:
            pending = None
            enqueue(0, starts[0])
            for ci, r0 in enumerate(starts):
                i = ci & 1
                if ci + 1 < len(starts):
                    if pending is not None:          # the other buffer must be drained first
                        for f in pending:
                            f.result()
                        pending = None
                    enqueue(i ^ 1, starts[ci + 1])
                events[i].synchronize()
                r1 = min(rows, r0 + chunk)
                src = stages[i].numpy()[:r1 - r0]
                if pending is not None:
                    for f in pending:
                        f.result()
                step = max(1, (r1 - r0 + nthr - 1) // nthr)
                pending = [pool.submit(move, out[r0 + s:min(r1, r0 + s + step)], src[s:s + step])
                           for s in range(0, r1 - r0, step)]
            if pending is not None:
                for f in pending:
                    f.result()
        return out

    @property
    def Z(self):
        if self._Z is None:
            self._Z = self._stack(self._zb, self._n, self.r)
        return self._Z

    @property
    def Y(self):
        if self._Y is None:
            self._Y = self._stack(self._yb, self._m, self.r)
        return self._Y

    @property
    def device_blocks(self):
        return self._zb, self._yb

    @property
    def steps(self):
        return len(self.gammas)

    @property
    def col_dim(self):
        return self.steps * self.r

    def gamma_diag(self):
        return np.repeat(np.asarray(self.gammas, dtype=complex), self.r)

    def dense(self):
        if self.col_dim == 0:
            return np.zeros((self.Z.shape[0], self.Y.shape[0]), dtype=complex)
        return (self.Z * self.gamma_diag()[None, :]) @ self.Y.conj().T


@dataclass
class AdiState:
    """adi.py:295-342 (w, t, u, v, factors and histories after the run)."""
    k: int
    Z: object
    Y: object
    gammas: list
    w: np.ndarray
    t: np.ndarray
    u: float
    v: float
    shift_history: list
    inner_residuals_A: list
    inner_residuals_B: list
    keep_inner_residuals: bool
    #: device-resident runs: the z_k / y_k blocks (Z / Y stay None until asked)
    z_blocks: list = None
    y_blocks: list = None

    def solution(self, r):
        return LowRankSolution(Z=self.Z, gammas=self.gammas, Y=self.Y, r=r)

    @staticmethod
    def _hstack(blocks, rows):
        if not blocks:
            return np.zeros((rows, 0), dtype=complex)
        if hasattr(blocks[0], "data_ptr"):            # device blocks
            return LowRankSolution._stack(list(blocks), rows, blocks[0].shape[1])
        return np.hstack(blocks)

    def S_A(self):
        """adi.py:334-337 (device blocks are downloaded)."""
        if not self.keep_inner_residuals:
            raise ValueError("inner residual blocks were not retained")
        return self._hstack(self.inner_residuals_A, self.w.shape[0])

    def S_B(self):
        """adi.py:339-342."""
        if not self.keep_inner_residuals:
            raise ValueError("inner residual blocks were not retained")
        return self._hstack(self.inner_residuals_B, self.t.shape[0])


# -- the paper's tolerance strategies (host scalars) --------------------------

def tolerance_budget(config, k, u_prev=0.0, v_prev=0.0, gap_budget=None):
    """Per-step budget for psi(||r^A||, ||r^B||): eps-hat^(1) spreads the gap
    budget uniformly (PAPER Eq. 30); back-looking strategies use eps-hat^(2),
    crediting unused allowance through u, v (Eq. 33).  adi.py:347-361."""
    eps = config.gap_budget if gap_budget is None else gap_budget
    if eps is None:
        raise ValueError("gap budget is not set")
    if _strategy(config.strategy) in _BACK_LOOKING:
        allowance = config.xi * k * eps / (2.0 * C_BOUND * config.kmax)
        return abs(allowance - u_prev - v_prev) / C_BOUND
    return config.xi * eps / (2.0 * C_BOUND ** 2 * config.kmax)


def tolB_from_tolA(delta_A, eps_check, c_check, norm_t, norm_w):
    """Boundary of the admissible region, clipped at 0 (adi.py:364-369)."""
    return max((eps_check - c_check * delta_A * norm_t) /
               (c_check * (2.0 * delta_A + norm_w)), 0.0)


def choose_tolerances(config, k, norm_w, norm_t, eps_hat):
    """Admissible (delta_A, delta_B) for the budget (adi.py:372-408; PAPER
    Eqs. 34-36)."""
    s = _strategy(config.strategy)
    if s is Strategy.EXACT_DIRECT:
        return ToleranceDecision(0.0, 0.0, eps_hat, s)
    if s is Strategy.FIXED:
        return ToleranceDecision(config.fixed_delta, config.fixed_delta, eps_hat, s)
    tiny = 1e-300
    if s is Strategy.DIRECT_A_ITER_B:
        raw = eps_hat / max(norm_w, tiny)
        return ToleranceDecision(0.0, min(max(raw, config.delta_min_B), config.delta_max_B),
                                 eps_hat, s, clamped_B_min=raw < config.delta_min_B)
    if s is Strategy.ITER_A_DIRECT_B:
        raw = eps_hat / max(norm_t, tiny)
        return ToleranceDecision(min(max(raw, config.delta_min_A), config.delta_max_A), 0.0,
                                 eps_hat, s, clamped_A_min=raw < config.delta_min_A)
    if s in (Strategy.DYNAMIC_MID, Strategy.DYNAMIC_MID_BL):
        mid = 0.5 * (min(config.delta_max_A, eps_hat / max(norm_t, tiny)) - config.delta_min_A)
        dA = max(mid, config.delta_min_A)
        rawB = (eps_hat - dA * norm_t) / (2.0 * dA + norm_w)
        dB = max(min(rawB, config.delta_max_B), config.delta_min_B)
        return ToleranceDecision(dA, dB, eps_hat, s, clamped_A_min=mid < config.delta_min_A,
                                 clamped_B_min=rawB < config.delta_min_B)
    dB = config.delta_min_B
    rawA = (eps_hat - dB * norm_w) / (norm_t + 2.0 * dB)
    dA = max(min(rawA, config.delta_max_A), config.delta_min_A)
    return ToleranceDecision(dA, dB, eps_hat, s, clamped_A_min=rawA < config.delta_min_A)


# -- drivers ------------------------------------------------------------------------

def run(problem, config, shift_sequence, bindings=None, **kw):
    """(LowRankSolution, SolveReport) -- adi.py:540-550."""
    sol, rep, _ = run_with_state(problem, config, shift_sequence, bindings=bindings, **kw)
    return sol, rep


def run_with_state(problem, config, shift_sequence, bindings=None, *, restart=50,
                   flexible=False, device=0, concurrent="auto", keep_on_device=False,
                   engine="auto", solver="gmres"):
    """adi.py:553-607.  ``bindings=None`` runs the device-resident driver with
    GpuGmresBinding(restart, flexible) on both sides; otherwise the host loop
    drives the given bindings."""
    if not isinstance(problem, SylvesterProblem):
        problem = SylvesterProblem.from_reference(problem)
    if not isinstance(config, AdiConfig):
        config = _adopt_config(config)
    if bindings is not None:
        return _run_host(problem, config, shift_sequence, bindings)
    return _run_device(problem, config, shift_sequence, restart=restart, flexible=flexible,
                       device=device, concurrent=concurrent, keep_on_device=keep_on_device,
                       engine=engine, solver=solver)


def _adopt_config(cfg):
    names = AdiConfig.__dataclass_fields__.keys()
    kw = {k: getattr(cfg, k) for k in names if hasattr(cfg, k)}
    return AdiConfig(**kw)


def _run_host(problem, config, shifts, bindings):
    """The reference's host loop (adi.py:510-607) around arbitrary bindings."""
    t0 = time.perf_counter()
    r = problem.r
    w = problem.f.astype(complex)
    t = problem.g.astype(complex)
    Zs, Ys, gammas, hist, SA, SB = [], [], [], [], [], []
    u = v = 0.0
    res0 = problem.rhs_norm()
    report = SolveReport(rhs_norm=res0, strategy=config.strategy)
    if res0 == 0.0:
        report.converged = True
        report.final_scaled_residual = 0.0
        state = AdiState(0, np.zeros((problem.n, 0), complex), np.zeros((problem.m, 0), complex),
                         [], w, t, 0.0, 0.0, [], [], [], config.keep_inner_residuals)
        return state.solution(r), report, state
    gap = config.gap_budget if config.gap_budget is not None else config.outer_tolerance * res0
    CT = None if problem.C is None else problem.C.T.tocsr()
    res = res0
    k_done = 0
    for k in range(1, config.kmax + 1):
        ts = time.perf_counter()
        eps_hat = tolerance_budget(config, k, u, v, gap)
        dec = choose_tolerances(config, k, block_norm(w), block_norm(t), eps_hat)
        alpha, beta = (complex(s) for s in shifts.at(k))
        ra = bindings.A.solve(beta, w, dec.delta_A if dec.delta_A > 0 else 1.0)
        rb = bindings.B.solve(alpha, t, dec.delta_B if dec.delta_B > 0 else 1.0)
        z, y = ra.solution, rb.solution
        gam = gamma(alpha, beta)
        Mz = z if problem.M is None else problem.M @ z
        Cty = y if CT is None else CT @ y
        rA, rB = ra.block_residual_norm, rb.block_residual_norm
        w = w + gam * Mz
        t = t + np.conj(gam) * Cty
        u += abs(gam) * block_norm(Mz) * rB
        v += abs(gam) * block_norm(Cty) * rA
        Zs.append(z)
        Ys.append(y)
        gammas.append(gam)
        hist.append((alpha, beta))
        if config.keep_inner_residuals:
            SA.append(ra.residual)
            SB.append(rb.residual)
        k_done = k
        res = computed_residual_norm(w, t)
        report.records.append(_record(k, res / res0, dec, rA, rB, ra, rb, u, v,
                                      1000.0 * (time.perf_counter() - ts)))
        if res < config.outer_tolerance * res0:
            break
    report.converged = bool(res < config.outer_tolerance * res0)
    report.outer_iterations = k_done
    report.final_scaled_residual = res / res0
    report.wall_ms = 1000.0 * (time.perf_counter() - t0)
    Z = np.hstack(Zs) if Zs else np.zeros((problem.n, 0), complex)
    Y = np.hstack(Ys) if Ys else np.zeros((problem.m, 0), complex)
    state = AdiState(k_done, Z, Y, gammas, w, t, u, v, hist, SA, SB, config.keep_inner_residuals)
    return state.solution(r), report, state


def _record(k, scaled, dec, rA, rB, ra, rb, u, v, wall_ms):
    rec = StepRecord(step=k, scaled_res=scaled, delta_A=dec.delta_A, delta_B=dec.delta_B,
                     achieved_rA=rA, achieved_rB=rB, inner_it_A=ra.total_iterations,
                     inner_it_B=rb.total_iterations, u=u, v=v, wall_ms=wall_ms,
                     a_converged=bool(np.all(ra.converged)),
                     b_converged=bool(np.all(rb.converged)),
                     clamped_A_min=dec.clamped_A_min, clamped_B_min=dec.clamped_B_min)
    if not (rec.a_converged and rec.b_converged):
        warnings.warn(f"inner solver missed its target at step {k}; "
                      "continuing with the achieved residual")
    return rec


#: largest A-side block (n x r complex128 bytes) for which the A and B solves
#: run concurrently by default (DeviceAdi(concurrent="auto"))
CONCURRENT_MAX_BLOCK_BYTES = 16 << 20
#: engine="auto": the ring multi-kernel engine when both sides' blocks are at least this large
AUTO_RING_BLOCK_BYTES = 192 << 20


class DeviceAdi:
    """Device-resident ADI engine: uploads once, then ``run()`` may be repeated
    (the bench times repeated runs with the inputs already in HBM)."""

    def __init__(self, problem, config, shift_sequence, *, restart=50, flexible=False,
                 device=0, concurrent="auto", engine="auto", phase_a="auto",
                 row_ranks=1, solver="gmres", native="auto", sm_split=None):
        import torch
        if not isinstance(problem, SylvesterProblem):
            problem = SylvesterProblem.from_reference(problem)
        if not isinstance(config, AdiConfig):
            config = _adopt_config(config)
        for side in ("A", "B"):
            if config.side_mode(side) != "iterative":
                raise NotImplementedError(
                    f"{config.strategy.value}: direct inner solves are not on the GPU hot path")
        self.problem, self.config, self.shifts = problem, config, shift_sequence
        self.device = device
        if engine == "auto":
            # Both sides HBM-bound and large (config 5: 512 / 262 MB blocks): the
            # multi-kernel delayed-Gram engine -- stand-alone banded SpMM and the
            # basis sweeps through a TMA ring, one slab per side -- beats the
            # persistent kernel, whose in-kernel SpMM sub-phase shares the block's
            # shared memory with the sweeps (config 5: 39.4 s vs 44.2 s).  Smaller
            # blocks are bound by per-step latency: one persistent launch per solve
            # (config 3: 16.4 s vs 17.9 s; config 2: 0.07 s vs 0.36 s).
            big = min(problem.n, problem.m) * problem.r * 16 >= AUTO_RING_BLOCK_BYTES
            engine = "rowpart" if (big and solver == "gmres" and problem.r <= 8) else "persistent"
        self.engine = engine
        self.solver = solver
        # the outer loop in native code (sad_adi_run) for the persistent GMRES
        # engine; the Python loop below stays the reference implementation
        # (keep_inner_residuals: the Python loop retains each step's inner
        # residual blocks, adi.py:533-535; the native loop reuses one buffer)
        self.native = (native is True or native == "auto") and engine == "persistent" \
            and solver == "gmres" and row_ranks == 1 and problem.r <= 8 \
            and _strategy(config.strategy).value in _lib.STRATEGY_CODES \
            and not config.keep_inner_residuals
        if native is True and not self.native:
            raise ValueError("native outer loop needs the persistent GMRES engine, r <= 8, "
                             "an iterative strategy and keep_inner_residuals=False")
        if concurrent == "auto":
            # Small blocks are latency-bound: the two solves overlap on disjoint
            # SM sets.  Large blocks are HBM-bound: one solve at a time on every
            # SM (no idle SMs while the shorter side waits for the longer one).
            concurrent = problem.n * problem.r * 16 <= CONCURRENT_MAX_BLOCK_BYTES
        self.concurrent = bool(concurrent)
        self.dev = torch.device("cuda", device)
        pairs = [shift_sequence.at(k) for k in range(1, min(config.kmax, _seq_len(shift_sequence)) + 1)]
        complex_run = (any(complex(a).imag != 0.0 or complex(b).imag != 0.0 for a, b in pairs)
                       or np.iscomplexobj(problem.f) or np.iscomplexobj(problem.g))
        self.tdtype = torch.complex128 if complex_run else torch.float64
        kind_a = config.precond_kind_A
        kind_b = config.precond_kind_B
        # concurrent A/B persistent solves: each side may occupy half of the SMs
        # (proportional to its size) so both cooperative grids are co-resident
        nsm = torch.cuda.get_device_properties(self.dev).multi_processor_count
        na, nb = problem.n, problem.m
        # SM share of the A side: the larger side also tends to need more Arnoldi
        # steps per solve, so the share is pushed past the row ratio (config 2:
        # rows 0.70 -> share 0.85, 77.4 -> 73.7 ms; tools/c2_split.py), clamped
        # so the smaller side keeps enough SMs
        if sm_split is None:
            frac_a = min(0.85, max(0.15, 0.5 + 2.0 * (na / (na + nb) - 0.5)))
        else:
            frac_a = float(sm_split)
        sm_a = max(1, min(nsm - 1, int(round(nsm * frac_a)))) if concurrent else 0
        sm_b = max(1, nsm - sm_a) if concurrent else 0
        if row_ranks > 1 or engine == "rowpart":
            # each side row-partitioned over `row_ranks` slabs, all ranks in this
            # process on one device (rowpart.py; the one-GPU test vehicle).
            # engine="rowpart" with one slab = the multi-kernel delayed-Gram engine
            # with the ring sweeps on the whole operator
            from .rowpart import RowPartitionedGmres
            self.concurrent = False
            self._pool = None
            mk = dict(max_iterations=config.max_inner_iterations, restart=restart,
                      flexible=flexible, device=device, nranks=row_ranks, comm="local")
            self.bA = RowPartitionedGmres("A", problem.A, problem.M, "iterative", kind_a, **mk)
            self.bB = RowPartitionedGmres("B", problem.B, problem.C, "iterative", kind_b, **mk)
            self._init_tail(problem)
            return
        self.bA = GpuGmresBinding("A", problem.A, problem.M, "iterative", kind_a,
                                  config.precond_droptol_A,
                                  max_iterations=config.max_inner_iterations, restart=restart,
                                  flexible=flexible, device=device, engine=engine,
                                  max_sms=sm_a, phase_a=phase_a, solver=solver)
        self.bB = GpuGmresBinding("B", problem.B, problem.C, "iterative", kind_b,
                                  config.precond_droptol_B,
                                  max_iterations=config.max_inner_iterations, restart=restart,
                                  flexible=flexible, device=device, engine=engine,
                                  max_sms=sm_b, phase_a=phase_a, solver=solver)
        self._pool = ThreadPoolExecutor(max_workers=2) if concurrent else None
        self._init_tail(problem)

    def _init_tail(self, problem):
        import torch
        self.Md = self.bA.mass      # M (for M z)
        self.Cd = self.bB.mass      # C with transpose (for C^T y)
        # upload in the host dtype, widen on the device
        self.f = torch.from_numpy(np.ascontiguousarray(problem.f)).to(self.dev).to(self.tdtype)
        self.g = torch.from_numpy(np.ascontiguousarray(problem.g)).to(self.dev).to(self.tdtype)
        self.sA = torch.cuda.Stream(device=self.dev)
        self.sB = torch.cuda.Stream(device=self.dev)
        self.h2d_bytes = (problem.f.nbytes + problem.g.nbytes)

    def warm(self):
        """Create the operators of every distinct shift and the workspaces."""
        for k in range(1, min(self.config.kmax, _seq_len(self.shifts)) + 1):
            a, b = self.shifts.at(k)
            self.bA.operator(b)
            self.bB.operator(a)

    def _native_fits(self):
        """z_k / y_k of every possible step preallocated as one buffer each:
        only when kmax steps fit in a quarter of the free device memory."""
        import torch
        esz = 16 if self.tdtype == torch.complex128 else 8
        need = self.config.kmax * (self.problem.n + self.problem.m) * self.problem.r * esz
        free, _ = torch.cuda.mem_get_info(self.dev)
        return need <= free // 4

    def _run_native(self, f=None, g=None):
        """DeviceAdi.run's loop in C++ (sad_adi_run): same steps, records and
        solution layout; the host does only scalar work between the solves."""
        import ctypes

        import torch
        cfg, prob = self.config, self.problem
        t0 = time.perf_counter()
        r, K = prob.r, cfg.kmax
        torch.cuda.synchronize(self.dev)
        w = (self.f if f is None else f).clone()
        t = (self.g if g is None else g).clone()
        dtype = _lib.SAD_F64 if self.tdtype == torch.float64 else _lib.SAD_C128
        pairs = [tuple(complex(x) for x in self.shifts.at(k)) for k in range(1, K + 1)]
        opsA = (ctypes.c_void_p * K)(*[self.bA.operator(b).handle.value for a, b in pairs])
        opsB = (ctypes.c_void_p * K)(*[self.bB.operator(a).handle.value for a, b in pairs])
        gam = np.array([gamma(a, b) for a, b in pairs], dtype=np.complex128)
        wsA = self.bA.workspace(r, dtype)
        wsB = self.bB.workspace(r, dtype)
        z_all = torch.empty((K, prob.n, r), dtype=self.tdtype, device=self.dev)
        y_all = torch.empty((K, prob.m, r), dtype=self.tdtype, device=self.dev)
        resA, resB = torch.empty_like(w), torch.empty_like(t)
        mz = torch.empty_like(w) if self.Md is not None else None
        cty = torch.empty_like(t) if self.Cd is not None else None
        c = _lib.AdiConfigC(
            strategy=_lib.STRATEGY_CODES[_strategy(cfg.strategy).value], kmax=K,
            max_inner_iterations=int(cfg.max_inner_iterations),
            outer_tolerance=cfg.outer_tolerance, xi=cfg.xi,
            gap_budget=0.0 if cfg.gap_budget is None else float(cfg.gap_budget),
            has_gap_budget=0 if cfg.gap_budget is None else 1,
            fixed_delta=cfg.fixed_delta, delta_min_A=cfg.delta_min_A, delta_max_A=cfg.delta_max_A,
            delta_min_B=cfg.delta_min_B, delta_max_B=cfg.delta_max_B)
        recs = np.zeros((K, _lib.SAD_ADI_REC), dtype=np.float64)
        summary = np.zeros(5, dtype=np.float64)
        steps = ctypes.c_int(0)
        cur = torch.cuda.current_stream(self.dev)
        self.sA.wait_stream(cur)
        self.sB.wait_stream(cur)
        ptr = lambda x: None if x is None else x.data_ptr()   # noqa: E731
        rc = _lib.load().sad_adi_run(
            _lib.context(self.device), ctypes.byref(c), r, dtype, prob.n, prob.m, wsA.handle,
            wsB.handle, opsA, opsB, gam.ctypes.data,
            None if self.Md is None else self.Md.handle, None if self.Cd is None else self.Cd.handle,
            w.data_ptr(), t.data_ptr(), z_all.data_ptr(), y_all.data_ptr(), resA.data_ptr(),
            resB.data_ptr(), ptr(mz), ptr(cty), 1 if self.concurrent else 0,
            ctypes.c_void_p(cur.cuda_stream), ctypes.c_void_p(self.sA.cuda_stream),
            ctypes.c_void_p(self.sB.cuda_stream), recs.ctypes.data, ctypes.byref(steps),
            summary.ctypes.data)
        _lib.check(rc, _lib.context(self.device))
        cur.wait_stream(self.sA)
        cur.wait_stream(self.sB)
        k_done = steps.value
        report = SolveReport(rhs_norm=float(summary[0]), strategy=cfg.strategy)
        for k in range(k_done):
            q = recs[k]
            rec = StepRecord(step=k + 1, scaled_res=q[0], delta_A=q[1], delta_B=q[2],
                             achieved_rA=q[3], achieved_rB=q[4], inner_it_A=int(q[5]),
                             inner_it_B=int(q[6]), u=q[7], v=q[8], wall_ms=q[13],
                             a_converged=bool(q[9]), b_converged=bool(q[10]),
                             clamped_A_min=bool(q[11]), clamped_B_min=bool(q[12]))
            if not (rec.a_converged and rec.b_converged):
                warnings.warn(f"inner solver missed its target at step {k + 1}; "
                              "continuing with the achieved residual")
            report.records.append(rec)
        report.converged = bool(summary[1])
        report.final_scaled_residual = float(summary[2]) if k_done else 0.0
        zb = [z_all[k] for k in range(k_done)]
        yb = [y_all[k] for k in range(k_done)]
        gammas = [complex(x) for x in gam[:k_done]]
        hist = pairs[:k_done]
        return self._finish(report, zb, yb, gammas, hist, w, t, float(summary[3]),
                            float(summary[4]), k_done, t0)

    def run(self, f=None, g=None):
        cyclic_ok = getattr(self.shifts, "cyclic", True) or \
            _seq_len(self.shifts) >= self.config.kmax
        if self.native and cyclic_ok and self._native_fits():
            return self._run_native(f, g)
        return self._run_python(f, g)

    def _run_python(self, f=None, g=None):
        import torch
        cfg, prob = self.config, self.problem
        t0 = time.perf_counter()
        r = prob.r
        torch.cuda.synchronize(self.dev)
        w = (self.f if f is None else f).clone()
        t = (self.g if g is None else g).clone()
        Gw, Gt = gram(w, device=self.device), gram(t, device=self.device)
        res0 = product_norm_from_grams(Gw, Gt)
        report = SolveReport(rhs_norm=res0, strategy=cfg.strategy)
        zb, yb, gammas, hist = [], [], [], []
        keep = bool(cfg.keep_inner_residuals)
        sa_blocks, sb_blocks = [], []
        u = v = 0.0
        if res0 == 0.0:
            report.converged = True
            report.final_scaled_residual = 0.0
            return self._finish(report, zb, yb, gammas, hist, w, t, u, v, 0, t0, keep=keep)
        gap = cfg.gap_budget if cfg.gap_budget is not None else cfg.outer_tolerance * res0
        res = res0
        k_done = 0
        solve_ms = 0.0
        for k in range(1, cfg.kmax + 1):
            ts = time.perf_counter()
            eps_hat = tolerance_budget(cfg, k, u, v, gap)
            dec = choose_tolerances(cfg, k, sigma_max_from_gram(Gw), sigma_max_from_gram(Gt),
                                    eps_hat)
            alpha, beta = (complex(s) for s in self.shifts.at(k))
            dA = dec.delta_A if dec.delta_A > 0 else 1.0
            dB = dec.delta_B if dec.delta_B > 0 else 1.0
            z = torch.empty_like(w)
            y = torch.empty_like(t)
            tsolve = time.perf_counter()
            ra, rb = self._solve_pair(beta, w, dA, z, alpha, t, dB, y)
            solve_ms += 1000.0 * (time.perf_counter() - tsolve)
            gam = gamma(alpha, beta)
            Mz = z if self.Md is None else self.Md.apply(z)
            Cty = y if self.Cd is None else self.Cd.apply(y, transpose=True)
            # one fused launch: w += gam Mz, t += conj(gam) C^T y and the six Grams
            G = adi_epilogue(gam, Mz, ra.residual, w, Cty, rb.residual, t, device=self.device)
            ra.residual_gram, rb.residual_gram = G[0], G[1]
            rA, rB = sigma_max_from_gram(G[0]), sigma_max_from_gram(G[1])
            u += abs(gam) * sigma_max_from_gram(G[2]) * rB
            v += abs(gam) * sigma_max_from_gram(G[3]) * rA
            zb.append(z)
            yb.append(y)
            gammas.append(gam)
            hist.append((alpha, beta))
            if keep:      # adi.py:533-535 (fresh device blocks every step)
                sa_blocks.append(ra.residual)
                sb_blocks.append(rb.residual)
            k_done = k
            Gw, Gt = G[4], G[5]
            res = product_norm_from_grams(Gw, Gt)
            report.records.append(_record(k, res / res0, dec, rA, rB, ra, rb, u, v,
                                          1000.0 * (time.perf_counter() - ts)))
            if res < cfg.outer_tolerance * res0:
                break
        report.converged = bool(res < cfg.outer_tolerance * res0)
        report.final_scaled_residual = res / res0
        report.device_timing["inner_solve_ms"] = solve_ms
        return self._finish(report, zb, yb, gammas, hist, w, t, u, v, k_done, t0,
                            keep=keep, sa=sa_blocks, sb=sb_blocks)

    def _solve_pair(self, beta, w, dA, z, alpha, t, dB, y):
        import torch
        if self._pool is None:
            ra = self.bA.solve_device(beta, w, dA, x=z)
            rb = self.bB.solve_device(alpha, t, dB, x=y)
            return ra, rb
        cur = torch.cuda.current_stream(self.dev)
        self.sA.wait_stream(cur)
        self.sB.wait_stream(cur)
        if self.engine == "persistent" and self.solver == "gmres" and w.shape[1] <= 8:
            # both persistent solves in flight from this thread, one wait each
            resA = torch.empty_like(w)
            resB = torch.empty_like(t)
            ta = self.bA.begin_device(beta, w, dA, z, resA, self.sA)
            tb = self.bB.begin_device(alpha, t, dB, y, resB, self.sB)
            ra, rb = self.bA.end_device(ta), self.bB.end_device(tb)
            cur.wait_stream(self.sA)
            cur.wait_stream(self.sB)
            return ra, rb

        def side(binding, stream, shift, rhs, delta, x):
            with torch.cuda.device(self.dev):
                return binding.solve_device(shift, rhs, delta, x=x, stream=stream)

        fa = self._pool.submit(side, self.bA, self.sA, beta, w, dA, z)
        fb = self._pool.submit(side, self.bB, self.sB, alpha, t, dB, y)
        ra, rb = fa.result(), fb.result()
        cur.wait_stream(self.sA)
        cur.wait_stream(self.sB)
        return ra, rb

    def _finish(self, report, zb, yb, gammas, hist, w, t, u, v, k_done, t0, keep=False,
                sa=(), sb=()):
        import torch
        torch.cuda.synchronize(self.dev)
        report.outer_iterations = k_done
        report.wall_ms = 1000.0 * (time.perf_counter() - t0)
        sol = LowRankSolution(gammas=gammas, r=self.problem.r, z_blocks=zb, y_blocks=yb,
                              n=self.problem.n, m=self.problem.m)
        state = AdiState(k_done, None, None, gammas, w, t, u, v, hist, list(sa), list(sb),
                         bool(keep), z_blocks=zb, y_blocks=yb)
        return sol, report, state


def _seq_len(seq):
    try:
        return len(seq)
    except TypeError:
        return len(seq.pairs)


def _run_device(problem, config, shifts, restart, flexible, device, concurrent,
                keep_on_device, engine="auto", solver="gmres"):
    t0 = time.perf_counter()
    eng = DeviceAdi(problem, config, shifts, restart=restart, flexible=flexible,
                    device=device, concurrent=concurrent, engine=engine, solver=solver)
    t1 = time.perf_counter()
    sol, rep, state = eng.run()
    for b in (eng.bA, eng.bB):      # workspaces back to the pool before the next run
        if hasattr(b, "release"):
            b.release()
    t2 = time.perf_counter()
    if not keep_on_device:
        state.Z, state.Y = sol.Z, sol.Y
        state.z_blocks = state.y_blocks = None
        state.w = state.w.cpu().numpy().astype(complex)
        state.t = state.t.cpu().numpy().astype(complex)
        state.inner_residuals_A = [b.cpu().numpy().astype(complex) for b in state.inner_residuals_A]
        state.inner_residuals_B = [b.cpu().numpy().astype(complex) for b in state.inner_residuals_B]
    rep.device_timing.update(construct_ms=1e3 * (t1 - t0), run_ms=1e3 * (t2 - t1),
                             download_ms=1e3 * (time.perf_counter() - t2))
    return sol, rep, state
