"""Golden fixtures for the incomplete-factorisation preconditioners (build
container only: runs the REFERENCE).

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_precond.py

Imports ``sylvadi`` from /root/reference/pkg/src (read-only) and writes

* tests/golden/ref_precond.npz -- for seeded small shifted operators (2-D
  convection-diffusion 12 x 12 and 24 x 24, its adjoint side, a complex shift,
  the symmetric Laplacian in the positive- and negative-definite range, a
  generalised pencil A + s M): the reference's factors (``factorize``,
  precond.py:307-357: ilu0 / ilut / ic0 / ict; L, U or G as raw CSR triplets),
  ``apply`` and ``apply_spd`` on a seeded complex block (precond.py:224-256),
  the breakdown cases (zero pivot, indefinite matrix for the Cholesky kinds),
  and the reference's BiCGstab / MINRES runs preconditioned with them
  (krylov.py:160-184, 271-287: iterations, solution, residual norms);
* tests/golden/ref_c1_ilut_bicgstab.csv, ref_c1_ilu0_bicgstab.csv -- per-step
  records of the reference's run_with_state on config 1 with its own
  ILUT(0.1) / ILU0-BiCGstab inner path (the paper's preconditioner,
  PAPER.md:638-649);
* tests/golden/ref_sym_ict_minres.csv -- the symmetric Laplacian pair of
  make_golden_minres.py with ICT(0.1)-MINRES on both sides.

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
from sylvadi import precond as rp  # noqa: E402
from sylvadi.problems import ConvDiffSpec, convdiff_matrix, random_rhs  # noqa: E402
from sylvadi.sparse import ShiftedOperator, SparseMatrix  # noqa: E402

sys.path.insert(0, os.path.join(REPO, "tests", "golden"))
from make_golden import write_csv  # noqa: E402

from paper_2312_02891_b200 import configs as cfgs  # noqa: E402

GOLD = os.path.join(REPO, "tests", "golden")


def put_csr(data, key, mat):
    m = sp.csr_matrix(mat.scipy() if hasattr(mat, "scipy") else mat)
    m.sort_indices()
    data[key + "_indptr"] = m.indptr.astype(np.int64)
    data[key + "_indices"] = m.indices.astype(np.int64)
    data[key + "_data"] = m.data
    data[key + "_n"] = np.array([m.shape[0]])


def factor_case(data, name, base, mass, shift, kind, droptol, x, adjoint=False):
    """factorize + apply (+ apply_spd) of the reference on one shifted operator."""
    op = ShiftedOperator(base, mass, shift, adjoint=adjoint)
    fact = rp.factorize(op.assembled(), kind, droptol=droptol, shift=shift)
    data[f"{name}_kind"] = np.array([kind])
    data[f"{name}_droptol"] = np.array([droptol])
    data[f"{name}_shift"] = np.array([complex(shift)])
    data[f"{name}_adjoint"] = np.array([adjoint])
    if kind in ("ilu0", "ilut"):
        for k, arr in zip(("li", "lj", "lv", "ui", "uj", "uv"), fact._lu):
            data[f"{name}_{k}"] = np.asarray(arr)
    else:
        for k, arr in zip(("gi", "gj", "gv"), fact._chol):
            data[f"{name}_{k}"] = np.asarray(arr)
        data[f"{name}_sign"] = np.array([fact.sign])
        data[f"{name}_apply_spd"] = fact.apply_spd(x)
    data[f"{name}_apply"] = fact.apply(x)
    nnz = (fact._lu[2].size + fact._lu[5].size) if fact._lu is not None else fact._chol[2].size
    print(f"{name}: {kind}({droptol}) factor nnz {nnz}")
    return op, fact


def solve_case(data, name, op, fact, b, delta, solver, maxit=1000):
    req = rk.InnerSolveRequest(op, b, delta, max_iterations=maxit, preconditioner=fact)
    res = rk.minres(req) if solver == "minres" else rk.bicgstab(req)
    data[f"{name}_{solver}_b"] = b
    data[f"{name}_{solver}_delta"] = np.array([delta])
    data[f"{name}_{solver}_x"] = res.solution
    data[f"{name}_{solver}_iters"] = res.iterations
    data[f"{name}_{solver}_norms"] = res.achieved_residual_norms
    data[f"{name}_{solver}_conv"] = res.converged
    print(f"  {solver}: iters {res.iterations} norms {res.achieved_residual_norms}")


def main():
    data = {}
    rng = np.random.default_rng(11)
    cd12 = convdiff_matrix(ConvDiffSpec(2, 12, (lambda x, y: 10.0 * x, lambda x, y: 10.0 * y)))    # n = 144
    cd24 = convdiff_matrix(ConvDiffSpec(2, 24, (lambda x, y: 50.0 * y, lambda x, y: -50.0 * x)))   # n = 576
    lap16 = convdiff_matrix(ConvDiffSpec(2, 16, None))            # n = 256, symmetric, negative definite
    put_csr(data, "cd12", cd12)
    put_csr(data, "cd24", cd24)
    put_csr(data, "lap16", lap16)
    x12 = rng.standard_normal((144, 3)) + 1j * rng.standard_normal((144, 3))
    x24 = rng.standard_normal((576, 2)) + 1j * rng.standard_normal((576, 2))
    x16 = rng.standard_normal((256, 2)) + 1j * rng.standard_normal((256, 2))
    data["x12"], data["x24"], data["x16"] = x12, x24, x16
    b12 = rng.standard_normal((144, 2))
    b24 = rng.standard_normal((576, 2))
    b16 = rng.standard_normal((256, 2))
    names = []

    def fc(name, *a, **k):
        names.append(name)
        return factor_case(data, name, *a, **k)

    # unsymmetric, real shift: the four ILU settings
    for kind, tol in (("ilu0", 0.0), ("ilut", 0.1), ("ilut", 0.01), ("ilut", 1e-4)):
        nm = f"cd12_{kind}_{tol:g}"
        op, fact = fc(nm, cd12, None, -30.0, kind, tol, x12)
        solve_case(data, nm, op, fact, b12, 1e-8, "bicgstab")
    # larger, B side (adjoint operator), real shift
    for kind, tol in (("ilu0", 0.0), ("ilut", 0.01)):
        nm = f"cd24adj_{kind}_{tol:g}"
        op, fact = fc(nm, cd24, None, -100.0, kind, tol, x24, adjoint=True)
        solve_case(data, nm, op, fact, b24, 1e-8, "bicgstab")
    # complex shift (complex factors), both sides
    op, fact = fc("cd12_c_ilut", cd12, None, -30.0 + 40.0j, "ilut", 0.01, x12)
    solve_case(data, "cd12_c_ilut", op, fact, b12, 1e-8, "bicgstab")
    op, fact = fc("cd24adj_c_ilu0", cd24, None, -100.0 - 75.0j, "ilu0", 0.0, x24, adjoint=True)
    solve_case(data, "cd24adj_c_ilu0", op, fact, b24, 1e-8, "bicgstab")
    # symmetric negative definite (negated before the Cholesky process): MINRES + BiCGstab
    for kind, tol in (("ic0", 0.0), ("ict", 0.1), ("ict", 0.01)):
        nm = f"lap16_{kind}_{tol:g}"
        op, fact = fc(nm, lap16, None, -10.0, kind, tol, x16)
        solve_case(data, nm, op, fact, b16, 1e-8, "minres")
        solve_case(data, nm, op, fact, b16, 1e-8, "bicgstab")
    # positive definite: the negated Laplacian as the base
    pos = SparseMatrix(-lap16.scipy())
    put_csr(data, "pos16", pos)
    op, fact = fc("pos16_ict", pos, None, 25.0, "ict", 0.02, x16)
    solve_case(data, "pos16_ict", op, fact, b16, 1e-9, "minres")
    # generalised pencil A + s M (M SPD, tridiagonal)
    n = 144
    m = sp.diags([np.full(n - 1, 1.0), np.full(n, 4.0), np.full(n - 1, 1.0)], [-1, 0, 1]).tocsr() / 6.0
    put_csr(data, "mass12", m)
    op, fact = fc("cd12_pencil_ilut", cd12, SparseMatrix(m), -45.0, "ilut", 0.01, x12)
    solve_case(data, "cd12_pencil_ilut", op, fact, b12, 1e-8, "bicgstab")
    op, fact = fc("cd12_pencil_adj_c_ilu0", cd12, SparseMatrix(m), -45.0 + 10.0j, "ilu0", 0.0, x12,
                  adjoint=True)
    solve_case(data, "cd12_pencil_adj_c_ilu0", op, fact, b12, 1e-8, "bicgstab")
    data["cases"] = np.array(names)

    # breakdowns (precond.py:89-92, 285-286)
    z = sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]]))
    try:
        rp.factorize(SparseMatrix(z), "ilu0")
        raise AssertionError("expected a zero pivot")
    except rp.FactorizationBreakdown as exc:
        data["break_zero_pivot_msg"] = np.array([str(exc)])
    indef = SparseMatrix(lap16.scipy() + 500.0 * sp.eye(256, format="csr"))
    try:
        rp.factorize(indef, "ic0")
        raise AssertionError("expected an indefinite breakdown")
    except rp.FactorizationBreakdown as exc:
        data["break_indef_msg"] = np.array([str(exc)])
    np.savez_compressed(os.path.join(GOLD, "ref_precond.npz"), **data)
    print("wrote ref_precond.npz")

    # config 1 through the reference's own driver with its ILU-BiCGstab path
    A, B, M, Cm, f, g = cfgs.build_problem("c1")
    spec = cfgs.CONFIGS["c1"]
    pairs, cyclic = spec.load_shift_pairs()
    problem = sv.SylvesterProblem(A=SparseMatrix(A), B=SparseMatrix(B), f=f, g=g)
    seq = sv.ShiftSequence(pairs=pairs, cyclic=cyclic)
    for kind in ("ilut", "ilu0"):
        cfg = sv.AdiConfig(strategy="dynamic_mid_bl", kmax=150, precond_kind_A=kind,
                           precond_kind_B=kind, precond_droptol_A=0.1, precond_droptol_B=0.1)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            _, rep, _ = sv.run_with_state(problem, cfg, seq)
        write_csv(os.path.join(GOLD, f"ref_c1_{kind}_bicgstab.csv"), rep)
        print(kind, "steps", rep.outer_iterations, "converged", rep.converged,
              "inner", rep.sum_inner_A, rep.sum_inner_B)

    # symmetric pair with ICT(0.1)-MINRES (shifts of make_golden_minres.py)
    with open(os.path.join(GOLD, "ref_sym_shifts.json")) as fh:
        meta = json.load(fh)
    A = convdiff_matrix(ConvDiffSpec(2, meta["n0_A"], None))
    B = convdiff_matrix(ConvDiffSpec(2, meta["n0_B"], None))
    f, g = random_rhs(A.nrows, B.nrows, meta["r"], meta["seed"])
    problem = sv.SylvesterProblem(A=A, B=B, f=f, g=g)
    seq = sv.ShiftSequence(pairs=[tuple(p) for p in meta["pairs"]], cyclic=True)
    cfg = sv.AdiConfig(strategy="dynamic_mid_bl", kmax=meta["kmax"], precond_kind_A="ict",
                       precond_kind_B="ict", precond_droptol_A=0.1, precond_droptol_B=0.1)
    bind = sv.adi.make_bindings(problem, cfg)
    assert bind.A.uses_minres(meta["pairs"][0][1])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _, rep, _ = sv.run_with_state(problem, cfg, seq)
    write_csv(os.path.join(GOLD, "ref_sym_ict_minres.csv"), rep)
    print("ict steps", rep.outer_iterations, "converged", rep.converged,
          "inner", rep.sum_inner_A, rep.sum_inner_B)


if __name__ == "__main__":
    main()
