"""Golden fixtures for the device MINRES (build container only: runs the REFERENCE).

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_minres.py

Imports ``sylvadi`` from /root/reference/pkg/src (read-only) and writes:

* tests/golden/ref_minres.npz -- krylov.minres (krylov.py:187-287) on seeded
  Hermitian cases: the negated 2-D Laplacian (convdiff_matrix with omega = 0)
  on a 24 x 24 grid shifted into the definite and the indefinite range, with
  Jacobi (its SPD split |dinv|, precond.py:242-256) and without a
  preconditioner, real and complex right-hand sides, r = 1..3; the adjoint
  (B-side) operator; a generalised Hermitian pencil (A + s M, M the 5-point
  mass-like SPD matrix); plus the reference's own test_krylov.py cases;
* tests/golden/ref_sym_dynamic_mid_bl_minres.csv -- per-step records of the
  reference's run_with_state on a symmetric Sylvester pair (Laplacians
  32 x 32 / 24 x 24, r = 2, real heuristic shifts), where its SolverBinding
  dispatches every inner solve to MINRES (adi.py:468-488).

/root/reference is never read at test, smoke or bench time.
"""

import json
import os
import sys
import warnings

import numpy as np
import scipy.sparse as sp

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import sylvadi as sv  # noqa: E402  (the reference)
from sylvadi import krylov as rk  # noqa: E402
from sylvadi.problems import ConvDiffSpec, convdiff_matrix, random_rhs  # noqa: E402
from sylvadi.sparse import ShiftedOperator, SparseMatrix  # noqa: E402

sys.path.insert(0, os.path.join(REPO, "tests", "golden"))
from make_golden import write_csv  # noqa: E402

GOLD = os.path.join(REPO, "tests", "golden")


def lap(n0):
    return convdiff_matrix(ConvDiffSpec(dimension=2, n0=n0, omega=None))


def case(data, name, base, mass, shift, b, delta, precond, adjoint=False, maxit=1000):
    op = ShiftedOperator(base, mass, shift, adjoint=adjoint)
    fact = sv.factorize(op.assembled(), precond, shift=shift) if precond != "none" else None
    res = rk.minres(rk.InnerSolveRequest(op, b, delta, max_iterations=maxit,
                                         preconditioner=fact))
    data[f"{name}_base"] = base.scipy().toarray() if base.scipy().shape[0] <= 64 else np.zeros(0)
    data[f"{name}_shift"] = np.array([shift])
    data[f"{name}_b"] = b
    data[f"{name}_delta"] = np.array([delta])
    data[f"{name}_maxit"] = np.array([maxit])
    data[f"{name}_x"] = res.solution
    data[f"{name}_iters"] = res.iterations
    data[f"{name}_norms"] = res.achieved_residual_norms
    data[f"{name}_conv"] = res.converged
    print(name, "iters", res.iterations, "norms", res.achieved_residual_norms)


def main():
    data = {}
    rng = np.random.default_rng(7)
    A24 = lap(24)                       # n = 576, eigenvalues in (-4608, -39)
    n = A24.scipy().shape[0]
    meta = {"lap_n0": 24}
    b2 = rng.standard_normal((n, 2))
    b1c = rng.standard_normal((n, 1)) + 1j * rng.standard_normal((n, 1))
    b3 = rng.standard_normal((n, 3))
    # definite: A - 10 I (Jacobi, real rhs, r = 2)
    case(data, "def_jac", A24, None, -10.0, b2, 1e-8, "jacobi")
    # indefinite: A + 1500 I (crosses the spectrum)
    case(data, "indef_jac", A24, None, 1500.0, b2, 1e-7, "jacobi")
    # no preconditioner, complex rhs
    case(data, "def_none_c", A24, None, -3.0, b1c, 1e-9, "none")
    # adjoint (B side) with Jacobi, r = 3, iteration cap hit on purpose
    case(data, "adj_cap", A24, None, 800.0, b3, 1e-12, "jacobi", adjoint=True, maxit=40)
    # generalised Hermitian pencil A + s M, M SPD (tridiagonal-like mass)
    m = sp.diags([np.full(n - 1, 1.0), np.full(n, 4.0), np.full(n - 1, 1.0)],
                 [-1, 0, 1]).tocsr() / 6.0
    case(data, "pencil_jac", A24, SparseMatrix(m), -50.0, b2, 1e-8, "jacobi")
    data["pencil_mass"] = m.toarray()
    # the reference's own known answers (test_krylov.py:58-98)
    def dense_op(d):
        return ShiftedOperator(SparseMatrix(sp.csr_matrix(d)), None, 0.0)
    d = np.diag(-np.arange(1.0, 51.0))
    bb = rng.standard_normal((50, 1))
    r = rk.minres(rk.InnerSolveRequest(dense_op(d), bb, 1e-10))
    data["kat_diag_b"], data["kat_diag_x"], data["kat_diag_iters"] = bb, r.solution, r.iterations
    data["lap_A24"] = A24.scipy().toarray()
    np.savez_compressed(os.path.join(GOLD, "ref_minres.npz"), **data)
    print("wrote ref_minres.npz")

    # symmetric Sylvester pair: every inner solve goes to MINRES
    A = lap(32)
    B = lap(24)
    f, g = random_rhs(A.scipy().shape[0], B.scipy().shape[0], 2, 3)
    problem = sv.SylvesterProblem(A=A, B=B, f=f, g=g)
    ritzA = sv.shifts.pencil_ritz_sets(A, None, n_direct=10, n_inverse=20, source="A-side")
    ritzB = sv.shifts.pencil_ritz_sets(B, None, n_direct=10, n_inverse=20, source="B-side")
    pairs = list(sv.heuristic_shifts(ritzA, ritzB, npairs=8).pairs)
    assert all(complex(a).imag == 0.0 and complex(b_).imag == 0.0 for a, b_ in pairs), pairs
    seq = sv.ShiftSequence(pairs=pairs, cyclic=True)
    cfg = sv.AdiConfig(strategy="dynamic_mid_bl", kmax=100, precond_kind_A="jacobi",
                       precond_kind_B="jacobi")
    bind = sv.adi.make_bindings(problem, cfg)
    assert bind.A.symmetric and bind.B.symmetric and bind.A.uses_minres(pairs[0][0])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _, rep, _ = sv.run_with_state(problem, cfg, seq)
    write_csv(os.path.join(GOLD, "ref_sym_dynamic_mid_bl_minres.csv"), rep)
    with open(os.path.join(GOLD, "ref_sym_shifts.json"), "w") as fh:
        json.dump({"n0_A": 32, "n0_B": 24, "r": 2, "seed": 3, "kmax": 100,
                   "pairs": [[float(complex(a).real), float(complex(b_).real)] for a, b_ in pairs],
                   "meta": meta}, fh, indent=1)
    print("steps", rep.outer_iterations, "converged", rep.converged)


if __name__ == "__main__":
    main()
