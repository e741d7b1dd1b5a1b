"""Host-side logic of the reference's inner-solver dispatch (no GPU needed):
the symmetry test of SolverBinding (adi.py:413-419) and the solver argument
validation of GpuGmresBinding."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import sylvadi_oracle as orc
from paper_2312_02891_b200.krylov import SOLVERS, GpuGmresBinding, _side_symmetric
from paper_2312_02891_b200.problems import convdiff_fd


class _Wrapped:
    """Duck-typed stand-in for the reference's SparseMatrix (``.scipy()``)."""

    def __init__(self, m):
        self._m = m

    def scipy(self):
        return self._m


@pytest.mark.parametrize("omega,expect", [(None, True), ((10.0, 10.0), False)])
def test_side_symmetric_matches_oracle(omega, expect):
    A = convdiff_fd(2, 12, omega)
    assert _side_symmetric(A) is expect
    assert _side_symmetric(_Wrapped(A)) is expect
    assert orc.is_symmetric(A) is expect


def test_side_symmetric_tolerance():
    """adi.py:418-419: asymmetry below 1e-12 x max(|a_ij|, 1) still counts as
    symmetric."""
    A = convdiff_fd(2, 8).tolil()
    A[0, 1] = A[0, 1] * (1.0 + 1e-15)
    assert _side_symmetric(A.tocsr()) and orc.is_symmetric(A.tocsr())
    A[0, 1] = A[0, 1] + 1e-3
    assert not _side_symmetric(A.tocsr()) and not orc.is_symmetric(A.tocsr())


def test_solver_argument_validation():
    assert SOLVERS == ("gmres", "bicgstab", "minres", "reference")
    with pytest.raises(ValueError):
        GpuGmresBinding("A", sp.eye(4, format="csr"), None, solver="ilu-bicgstab")
    with pytest.raises(ValueError):
        GpuGmresBinding("C", sp.eye(4, format="csr"), None)
    with pytest.raises(NotImplementedError):
        GpuGmresBinding("A", sp.eye(4, format="csr"), None, mode="direct")


def test_oracle_reference_dispatch_on_pencils():
    """A symmetric base with a nonsymmetric mass is not a MINRES side."""
    A = convdiff_fd(2, 6)
    M = sp.eye(A.shape[0], format="csr") + sp.diags(np.full(A.shape[0] - 1, 0.1), 1, format="csr")
    b = orc.Binding("A", A, M, solver="reference")
    assert not b.uses_minres(-1.0)
    assert orc.Binding("A", A, sp.eye(A.shape[0], format="csr"), solver="reference").uses_minres(-1.0)
