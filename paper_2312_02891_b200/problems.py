"""Seeded test-problem generators for the BASELINE configurations.

Host-side harness code (not on the hot path).  The finite-difference
generator reproduces the reference's convection-diffusion matrices bit for bit
(``/root/reference/pkg/src/sylvadi/problems.py:52-91``: negated central FD,
``h = 1/(n0+1)``, first grid axis fastest) and ``random_rhs`` reproduces
``problems.py:105-118`` (Philox(seed) normals, g rescaled so that
||f||_F = ||g||_F).  Bit-equality with the reference is pinned by
``tests/test_problems.py`` against hashes recorded from the reference itself.

The bilinear-FEM generator (config 3) has no reference counterpart
(SURVEY.md D4): Q1 elements on the same interior grid and axis ordering,
stiffness + convection negated so that the pencil spectrum lies in C-.
"""

import numpy as np
import scipy.sparse as sp


def _grid_coords(dim, n0):
    h = 1.0 / (n0 + 1)
    n = n0 ** dim
    flat = np.arange(n)
    sub = np.empty((dim, n), dtype=np.int64)
    q = flat
    for ax in range(dim):
        q, sub[ax] = np.divmod(q, n0)
    return h, flat, sub, (sub + 1) * h


def convection_field(omega, coords):
    """Evaluate a convection spec (None, constants or callables) at points."""
    dim, npts = coords.shape
    if omega is None:
        return np.zeros((dim, npts))
    out = np.empty((dim, npts))
    for ax, comp in enumerate(omega):
        out[ax] = comp(*coords) if callable(comp) else float(comp)
    return out


def convdiff_fd(dim, n0, omega=None):
    """Negated central-difference matrix of ``-lap(u) + omega . grad(u)`` on
    the unit square/cube, homogeneous Dirichlet, ``n0`` interior points per
    axis (5-point in 2-D, 7-point in 3-D), canonical CSR (sorted, summed)."""
    if dim not in (2, 3):
        raise ValueError("dimension must be 2 or 3")
    if n0 < 1:
        raise ValueError("n0 must be >= 1")
    h, flat, sub, coords = _grid_coords(dim, n0)
    n = flat.size
    wind = convection_field(omega, coords)
    r_parts = [flat]
    c_parts = [flat]
    v_parts = [np.full(n, -2.0 * dim / h**2)]
    stride = 1
    for ax in range(dim):
        half = wind[ax] / (2.0 * h)
        up = sub[ax] < n0 - 1
        dn = sub[ax] > 0
        r_parts += [flat[up], flat[dn]]
        c_parts += [flat[up] + stride, flat[dn] - stride]
        v_parts += [(1.0 / h**2 - half)[up], (1.0 / h**2 + half)[dn]]
        stride *= n0
    mat = sp.coo_matrix((np.concatenate(v_parts),
                         (np.concatenate(r_parts), np.concatenate(c_parts))),
                        shape=(n, n)).tocsr()
    return canonical_csr(mat)


def canonical_csr(mat):
    """CSR with summed duplicates and sorted column indices (the invariants of
    the reference's SparseMatrix, sparse.py:39-53)."""
    csr = sp.csr_matrix(mat)
    csr.sum_duplicates()
    csr.sort_indices()
    if not np.all(np.isfinite(csr.data)):
        raise ValueError("matrix contains non-finite entries")
    return csr


def random_rhs(n, m, r, seed):
    """Philox(seed) normal factors f (n x r), g (m x r), g rescaled so that
    ||f||_F = ||g||_F (same generator calls, hence the same bits, as the
    reference's problems.py:105-118)."""
    if r < 1:
        raise ValueError("rhs rank must be >= 1")
    gen = np.random.Generator(np.random.Philox(seed))
    f = gen.standard_normal((n, r))
    g = gen.standard_normal((m, r))
    g *= np.linalg.norm(f) / np.linalg.norm(g)
    return f, g


def _q1_1d(n0):
    """1-D linear-element matrices on the interior nodes of (0, 1):
    mass h/6 [1 4 1], stiffness 1/h [-1 2 -1], convection phi_i phi_j' [-1/2 0 1/2]."""
    h = 1.0 / (n0 + 1)
    ones = np.ones(n0)
    off = np.ones(n0 - 1)
    mass = sp.diags([off * (h / 6.0), ones * (4.0 * h / 6.0), off * (h / 6.0)],
                    [-1, 0, 1], format="csr")
    stiff = sp.diags([-off / h, 2.0 * ones / h, -off / h], [-1, 0, 1], format="csr")
    conv = sp.diags([-0.5 * off, 0.5 * off], [-1, 1], format="csr")
    return mass, stiff, conv


def fem_q1_2d(n0, omega):
    """Bilinear (Q1) FEM pencil on an n0 x n0 interior grid of the unit square.

    Returns ``(A, M)`` with A = -(K + C): K the 9-point stiffness,
    C the 9-point convection (omega constant, 2 components) and M the 9-point
    consistent mass.  Axis 0 is fastest, so x-operators are the right Kronecker
    factor.  (New harness code: the reference has no FEM generator.)
    """
    m1, k1, c1 = _q1_1d(n0)
    wx, wy = float(omega[0]), float(omega[1])
    stiff = sp.kron(m1, k1) + sp.kron(k1, m1)
    conv = wx * sp.kron(m1, c1) + wy * sp.kron(c1, m1)
    A = canonical_csr(-(stiff + conv))
    M = canonical_csr(sp.kron(m1, m1))
    return A, M
