"""The GMRES restatement (new inner solver) on known answers (CPU)."""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import sylvadi_oracle as orc
from paper_2312_02891_b200 import configs as cfgs


def op_dense(d, shift=0.0, adjoint=False):
    return orc.ShiftedOp(sp.csr_matrix(d), None, shift, adjoint=adjoint)


def test_identity_one_iteration(rng):
    # analogue of test_krylov.py:15-20
    b = rng.standard_normal((6, 1))
    res = orc.gmres(op_dense(np.eye(6)), b, 1e-12, dinv=np.ones(6, complex))
    assert res.total_iterations <= 1
    assert np.max(np.abs(res.solution - b)) < 1e-12
    assert np.all(res.converged)


def test_loose_tolerance_zero_iterations(rng):
    # analogue of test_krylov.py:27-33
    b = rng.standard_normal((5, 1))
    res = orc.gmres(op_dense(np.eye(5)), b, 10.0 * np.linalg.norm(b))
    assert res.total_iterations == 0
    assert np.array_equal(res.solution, np.zeros((5, 1)))
    assert np.all(res.converged)


@pytest.mark.parametrize("flexible", [False, True])
@pytest.mark.parametrize("restart", [3, 10, 50])
def test_matches_dense_solve(rng, restart, flexible):
    n = 40
    d = rng.standard_normal((n, n)) + np.diag(np.abs(rng.standard_normal(n)) * 0 + 12.0)
    b = rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))
    op = op_dense(d, shift=-0.3 + 0.2j)
    res = orc.gmres(op, b, 1e-10, dinv=orc.jacobi_dinv(op), restart=restart,
                    flexible=flexible)
    assert np.all(res.converged)
    x = np.linalg.solve(d + (-0.3 + 0.2j) * np.eye(n), b)
    assert np.max(np.abs(res.solution - x)) <= 1e-9
    # achieved norms are true recomputed residuals (test_krylov.py:45-54)
    for c in range(3):
        check = np.linalg.norm(b[:, c] - (d + (-0.3 + 0.2j) * np.eye(n)) @ res.solution[:, c])
        assert abs(check - res.achieved_residual_norms[c]) <= 1e-13 * np.linalg.norm(b[:, c])
    assert np.all(res.achieved_residual_norms <= 1e-10 / 3)


def test_adjoint_side_matches_dense(rng):
    n = 30
    d = rng.standard_normal((n, n)) + 10 * np.eye(n)
    b = rng.standard_normal((n, 2))
    shift = -1.0 + 0.5j
    op = op_dense(d, shift, adjoint=True)
    res = orc.gmres(op, b, 1e-11, dinv=orc.jacobi_dinv(op), restart=7)
    x = np.linalg.solve((d + shift * np.eye(n)).conj().T, b)
    assert np.max(np.abs(res.solution - x)) <= 1e-9


def test_maxit_caps_iterations(rng):
    A, _, _, _, f, _ = cfgs.build_problem("c1")
    op = orc.ShiftedOp(A, None, -600.0)
    res = orc.gmres(op, f, 1e-14, max_iterations=7, dinv=orc.jacobi_dinv(op), restart=5)
    assert res.iterations[0] == 7
    assert not res.converged[0]


def test_solution_agrees_with_scipy_gmres():
    """Solutions (not counts: scipy is left-preconditioned MGS) agree."""
    A, _, _, _, f, _ = cfgs.build_problem("c1")
    shift = -637.2036526571874
    op = orc.ShiftedOp(A, None, shift)
    dinv = orc.jacobi_dinv(op)
    res = orc.gmres(op, f, 1e-9 * np.linalg.norm(f), dinv=dinv, restart=50)
    K = (A + shift * sp.eye(A.shape[0])).tocsc()
    x_ref = spla.spsolve(K, f[:, 0])
    rel = np.linalg.norm(res.solution[:, 0] - x_ref) / np.linalg.norm(x_ref)
    assert rel < 1e-6
    xs, info = spla.gmres(K, f[:, 0], rtol=1e-12, restart=50, maxiter=200)
    assert info == 0
    assert np.linalg.norm(xs - x_ref) / np.linalg.norm(x_ref) < 1e-6


def test_givens_zeroes_second_component(rng):
    for _ in range(20):
        f, g = rng.standard_normal(2) + 1j * rng.standard_normal(2)
        c, s, r = orc.givens(f, g)
        assert abs(c * f + s * g - r) < 1e-14 * (abs(f) + abs(g))
        assert abs(-np.conj(s) * f + c * g) < 1e-14 * (abs(f) + abs(g))
        assert abs(c * c + abs(s) ** 2 - 1.0) < 1e-14
