"""Shift sequences (``/root/reference/pkg/src/sylvadi/shifts.py:31-67``).

Shift generation itself (Ritz values + greedy heuristic) is outside the hot
path; shifts are pinned in JSON files in the reference's
own layout and read back here, so every run shares bit-identical shifts.
"""

import json
from dataclasses import dataclass


@dataclass
class ShiftSequence:
    pairs: list
    cyclic: bool = True

    def __post_init__(self):
        self.pairs = [(complex(a), complex(b)) for a, b in self.pairs]
        if not self.pairs:
            raise ValueError("shift sequence must not be empty")

    def __len__(self):
        return len(self.pairs)

    def at(self, k):
        """(alpha_k, beta_k) for 1-based outer step k, reused cyclically."""
        i = k - 1
        if i >= len(self.pairs):
            if not self.cyclic:
                raise IndexError("shift sequence exhausted")
            i %= len(self.pairs)
        return self.pairs[i]

    def to_json(self, path):
        with open(path, "w") as fh:
            json.dump({"cyclic": self.cyclic,
                       "pairs": [[[a.real, a.imag], [b.real, b.imag]] for a, b in self.pairs]},
                      fh, indent=1)

    @classmethod
    def from_json(cls, path):
        with open(path) as fh:
            payload = json.load(fh)
        return cls(pairs=[(complex(*a), complex(*b)) for a, b in payload["pairs"]],
                   cyclic=bool(payload.get("cyclic", True)))


# ---------------------------------------------------------------------------
# Shift generation: Ritz values on the device + the greedy
# picker on the host.  Same names, arguments and results as shifts.py:70-217;
# the sparse LU of the reference (splu, shifts.py:117-119) is replaced by the
# library's GMRES solves, so the inverse Ritz sets of configs 3-5 become
# feasible (splu would need weeks and terabytes at n = 8M).
# ---------------------------------------------------------------------------

import numpy as np  # noqa: E402

INF = float("inf")


@dataclass
class RitzSet:
    """shifts.py:18-28, plus ``bounds``: the Arnoldi residual norm
    |h_{k+1,k} e_k^T y| of each Ritz pair (None when unknown).  Only pairs with
    small bounds are determined by the operator; the others depend on rounding
    (and, for the inverse sets, on the solver), in the reference as here."""
    values: np.ndarray
    source: str
    kind: str
    bounds: np.ndarray = None

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.complex128).ravel()
        if not np.all(np.isfinite(self.values)):
            raise ValueError("Ritz values must be finite")


def arnoldi_ritz(apply, start, steps, source="A-side", kind="direct", device=0):
    """Ritz values of ``steps`` Arnoldi iterations (shifts.py:70-98) with the
    basis on the device.  ``apply(x)`` maps an (n, 1) complex128 device block
    to one; ``start`` is a host vector.  Modified Gram-Schmidt with one
    re-orthogonalisation pass in the reference's order, each inner product and
    update through the library (sad_gram / sad_axpy); breakdown when
    ``h_{j+1,j} < 1e-12 max(1, |h_jj|)`` returns the Ritz values found so far.
    """
    import torch
    from .device import axpy, gram
    v = np.asarray(start, dtype=np.complex128).ravel()
    nrm = np.linalg.norm(v)
    if nrm == 0.0:
        raise ValueError("Arnoldi start vector must be nonzero")
    if steps < 1:
        raise ValueError("steps must be >= 1")
    n = v.size
    steps = min(steps, n)
    dev = torch.device("cuda", device)
    V = [torch.from_numpy((v / nrm).reshape(n, 1)).to(dev)]
    H = np.zeros((steps + 1, steps), dtype=np.complex128)
    j = 0
    for j in range(steps):
        w = apply(V[j]).clone()
        for _ in range(2):
            for i in range(j + 1):
                h = complex(gram(V[i], w, device=device)[0, 0])
                H[i, j] += h
                axpy(-h, V[i], w, device=device)
        hn = float(np.sqrt(gram(w, device=device).real[0, 0]))
        H[j + 1, j] = hn
        if hn < 1e-12 * max(1.0, abs(H[j, j])):
            j += 1
            break
        nv = torch.zeros_like(w)
        axpy(1.0 / hn, w, nv, device=device)
        V.append(nv)
    else:
        j += 1
    theta, Yv = np.linalg.eig(H[:j, :j])
    bounds = np.abs(H[j, j - 1] * Yv[j - 1, :]) / np.linalg.norm(Yv, axis=0)
    return RitzSet(values=theta, source=source, kind=kind, bounds=bounds)


class _DeviceSolve:
    """x = Op^{-1} y for Op = base (shift 0) by the library's Jacobi-GMRES to a
    relative residual ``rtol`` (replaces splu(...).solve, shifts.py:117-129)."""

    def __init__(self, mat, rtol, restart, max_iterations, device):
        from .krylov import GpuGmresBinding
        self.binding = GpuGmresBinding("A", mat, None, precond_kind="jacobi", restart=restart,
                                       max_iterations=max_iterations, device=device)
        self.rtol = rtol
        self.device = device
        self.iterations = 0
        self.unconverged = 0

    def __call__(self, y):
        from .device import gram
        nrm = float(np.sqrt(gram(y, device=self.device).real[0, 0]))
        if nrm == 0.0:
            return y.clone()
        out = self.binding.solve_device(0.0, y, self.rtol * nrm)
        self.iterations += int(np.sum(out.iterations))
        self.unconverged += int(np.sum(~np.asarray(out.converged)))
        return out.solution


def pencil_ritz_sets(base, mass=None, n_direct=10, n_inverse=20, source="A-side", *,
                     rtol=1e-12, restart=50, max_iterations=20000, device=0, stats=None):
    """Direct and inverse Ritz sets of the pencil (base, mass) (shifts.py:101-129):
    Arnoldi on mass^{-1} base and on base^{-1} mass from a ones start vector;
    the inverse set holds the reciprocals.  Every operator action runs on the
    device; the solves are GMRES to ``rtol`` (``stats`` collects their
    iteration counts)."""
    from .device import DeviceMatrix
    Bd = DeviceMatrix(base, device=device)
    Md = None if mass is None else DeviceMatrix(mass, device=device)
    n = Bd.shape[0]
    start = np.ones(n)
    base_inv = _DeviceSolve(base, rtol, restart, max_iterations, device)
    mass_inv = None if mass is None else _DeviceSolve(mass, rtol, restart, max_iterations,
                                                      device)

    def direct_action(x):
        y = Bd.apply(x)
        return y if mass_inv is None else mass_inv(y)

    def inverse_action(x):
        y = x if Md is None else Md.apply(x)
        return base_inv(y)

    direct = arnoldi_ritz(direct_action, start, n_direct, source, "direct", device)
    inv = arnoldi_ritz(inverse_action, start, n_inverse, source, "inverse", device)
    keep = np.abs(inv.values) > 0
    inv_values = 1.0 / inv.values[keep]
    # relative bound of the reciprocal: |d(1/theta)| / |1/theta| = |d theta| / |theta|
    inv_bounds = inv.bounds[keep] / np.abs(inv.values[keep]) * np.abs(inv_values)
    if stats is not None:
        stats[source] = {"base_solve_iterations": base_inv.iterations,
                         "base_solve_unconverged": base_inv.unconverged,
                         "mass_solve_iterations": mass_inv.iterations if mass_inv else 0}
    return direct, RitzSet(values=inv_values, source=source, kind="inverse", bounds=inv_bounds)


def _merge(ritz):
    if isinstance(ritz, RitzSet):
        return ritz.values.copy()
    vals = [r.values if isinstance(r, RitzSet) else np.asarray(r, dtype=complex).ravel()
            for r in ritz]
    return np.concatenate(vals) if vals else np.empty(0, dtype=complex)


def shift_objective(alphas, betas, ritz_A, ritz_B):
    """max over Ritz pairs (lambda, mu) of prod_i |(lambda-a_i)(mu-b_i)| /
    |(lambda+b_i)(mu+a_i)|, INF when a denominator is within 1e-14 * scale of
    zero (shifts.py:141-164)."""
    lam, mu = _merge(ritz_A), _merge(ritz_B)
    alphas = np.asarray(alphas, dtype=complex).ravel()
    betas = np.asarray(betas, dtype=complex).ravel()
    if alphas.size != betas.size:
        raise ValueError("alpha and beta candidate sets must pair up")
    scale = max(np.abs(lam).max(initial=0.0), np.abs(mu).max(initial=0.0), 1.0)
    prod = np.ones((lam.size, mu.size))
    for a, b in zip(alphas, betas):
        dl, dm = np.abs(lam + b), np.abs(mu + a)
        if np.any(dl <= 1e-14 * scale) or np.any(dm <= 1e-14 * scale):
            return INF
        prod *= np.outer(np.abs(lam - a) / dl, np.abs(mu - b) / dm)
    return float(prod.max())


def heuristic_shifts(ritz_A, ritz_B, npairs=20):
    """Greedy Penzl-style pairs (shifts.py:167-217): candidates are the merged
    Ritz values with negative real part; each round takes the pair minimising
    (objective, |Im a| + |Im b|, |a| + |b|), first in (alpha, beta) candidate
    order on ties.  The objective of every candidate pair of a round is
    evaluated at once, with the reference's operation order per entry
    (prod * outer(u, v)), so the selection is bit-identical."""
    lam, mu = _merge(ritz_A), _merge(ritz_B)
    cand_a, cand_b = lam[lam.real < 0.0], mu[mu.real < 0.0]
    if cand_a.size == 0 or cand_b.size == 0:
        raise ValueError("no stable shift candidates in the Ritz sets")
    scale = max(np.abs(lam).max(), np.abs(mu).max(), 1.0)
    num_a = np.abs(lam[:, None] - cand_a[None, :])     # |lam - alpha|   (L, Na)
    den_b = np.abs(lam[:, None] + cand_b[None, :])     # |lam + beta|    (L, Nb)
    num_b = np.abs(mu[:, None] - cand_b[None, :])      # |mu - beta|     (Mu, Nb)
    den_a = np.abs(mu[:, None] + cand_a[None, :])      # |mu + alpha|    (Mu, Na)
    ok_a = np.all(den_a > 1e-14 * scale, axis=0)
    ok_b = np.all(den_b > 1e-14 * scale, axis=0)
    ia_ok, ib_ok = np.nonzero(ok_a)[0], np.nonzero(ok_b)[0]
    if ia_ok.size == 0 or ib_ok.size == 0:
        raise ValueError("all shift candidates hit a singular denominator")
    # tie-break keys of every (ia, ib), candidate order ia-major
    IA, IB = np.meshgrid(ia_ok, ib_ok, indexing="ij")
    key2 = (np.abs(cand_a.imag)[IA] + np.abs(cand_b.imag)[IB]).ravel()
    key3 = (np.abs(cand_a)[IA] + np.abs(cand_b)[IB]).ravel()
    u_all = num_a[:, IA] / den_b[:, IB]                # (L, na, nb)
    v_all = num_b[:, IB] / den_a[:, IA]                # (Mu, na, nb)
    prod = np.ones((lam.size, mu.size))
    pairs = []
    for _ in range(npairs):
        outer = u_all[:, None, :, :] * v_all[None, :, :, :]          # (L, Mu, na, nb)
        obj = (prod[:, :, None, None] * outer).max(axis=(0, 1)).ravel()
        best = np.lexsort((key3, key2, obj))[0]      # lexicographic, stable on full ties
        ia, ib = IA.ravel()[best], IB.ravel()[best]
        pairs.append((complex(cand_a[ia]), complex(cand_b[ib])))
        prod *= np.outer(num_a[:, ia] / den_b[:, ib], num_b[:, ib] / den_a[:, ia])
    return ShiftSequence(pairs=pairs, cyclic=True)
