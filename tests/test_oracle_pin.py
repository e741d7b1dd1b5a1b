"""Pin the CPU oracle against the reference (CPU only).

Fixtures in tests/golden/ were produced by running the reference itself
(tests/golden/make_golden.py); the known answers are the ones the reference's
own tests assert (file:line cited per test).
"""

import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import sylvadi_oracle as orc
from paper_2312_02891_b200 import configs as cfgs

from conftest import GOLD, read_steps_csv


@pytest.fixture(scope="module")
def small():
    return dict(np.load(os.path.join(GOLD, "ref_small.npz")))


# -- known answers from the reference's tests ----------------------------------

def test_budget_known_answer():
    # test_adi.py:47-52
    cfg = orc.Config(strategy="dynamic_mid", gap_budget=1e-8, kmax=50, xi=1.0)
    val = orc.tolerance_budget(cfg, 1)
    assert abs(val - 1e-8 / (2.0 * (6.0 + 4.0 * np.sqrt(2.0)) * 50)) < 1e-25
    assert abs(val - 8.5786e-12) < 1e-15 * 1e-12 + 1e-16


def test_bl_budget_exhausted():
    # test_adi.py:61-65
    eps = 1e-8
    cfg = orc.Config(strategy="dynamic_mid_bl", gap_budget=eps, kmax=50, xi=1.0)
    spent = 2.0 * eps / (2.0 * orc.C_BOUND * 50)
    assert orc.tolerance_budget(cfg, 2, spent, 0.0) == 0.0


def test_tolB_known_answer():
    # test_adi.py:84-88
    val = orc.tolB_from_tolA(1e-4, 1e-8, 3.0, 1e-5, 2e-3)
    assert abs(val - 1.0606e-6) < 1e-9


def test_dynamic_mid_worked_example():
    # test_adi.py:92-102
    cfg = orc.Config(strategy="dynamic_mid", delta_min_A=5e-10, delta_min_B=5e-10,
                     gap_budget=1.0)
    dA, dB, _, _ = orc.choose_tolerances(cfg, 2, 2e-3, 1e-5, 8.58e-12)
    assert abs(dA - 4.287e-7) < 1e-9
    assert abs(dB - 2.145e-9) < 2e-12


def test_residual_norm_known_answers(rng):
    # test_adi.py:28-37
    w = np.eye(3)[:, [0]]
    assert abs(orc.computed_residual_norm(w, 2.0 * w) - 2.0) < 1e-15
    q, _ = np.linalg.qr(rng.standard_normal((6, 2)))
    assert abs(orc.computed_residual_norm(q, q @ np.diag([3.0, 4.0])) - 4.0) < 1e-13


def test_jacobi_known_answer():
    # test_precond.py:105-108: Jacobi on diag(2,4) maps [2,4] to [1,1]
    op = orc.ShiftedOp(sp.diags([2.0, 4.0]).tocsr(), None, 0.0)
    d = orc.jacobi_dinv(op)
    assert np.allclose(d * np.array([2.0, 4.0]), [1.0, 1.0])


def test_scalar_step_known_answer():
    # test_adi.py:155-167: A=B=-1, M=C=1, f=g=1, shifts (-1,-1): z=-0.5, gamma=2, X=0.5
    one = sp.csr_matrix(np.array([[1.0]]))
    neg = sp.csr_matrix(np.array([[-1.0]]))
    op = orc.ShiftedOp(neg, one, -1.0)
    z = np.linalg.solve(op.apply(np.eye(1)), np.array([[1.0]]))
    assert abs(z[0, 0] + 0.5) < 1e-14
    assert orc.gamma(-1.0, -1.0) == 2.0


# -- reference outputs on seeded small cases --------------------------------------

@pytest.mark.parametrize("tag", ["real", "cplx"])
@pytest.mark.parametrize("adj", ["fwd", "adj"])
@pytest.mark.parametrize("mname", ["I", "M"])
def test_shifted_apply_matches_reference(small, tag, adj, mname):
    shift = {"real": -1.7 + 0j, "cplx": -2.0 + 0.4j}[tag]
    op = orc.ShiftedOp(sp.csr_matrix(small["base"]),
                       None if mname == "I" else sp.csr_matrix(small["mass"]),
                       shift, adjoint=(adj == "adj"))
    got = op.apply(small["x"])
    ref = small[f"apply_{tag}_{adj}_{mname}"]
    # test_sparse.py:99-106,116-124 tolerances
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    dref = small[f"dinv_{tag}_{adj}_{mname}"]
    assert np.max(np.abs(orc.jacobi_dinv(op) - dref)) <= 1e-15 * np.max(np.abs(dref))


def test_bicgstab_matches_reference(small):
    op = orc.ShiftedOp(sp.csr_matrix(small["bicg_dense"]), None, -0.5 + 0.25j)
    res = orc.bicgstab(op, small["bicg_b"], 1e-10, dinv=orc.jacobi_dinv(op))
    assert np.array_equal(res.iterations, small["bicg_iters"])
    assert np.max(np.abs(res.solution - small["bicg_x"])) <= 1e-12 * np.max(np.abs(small["bicg_x"]))
    assert np.all(res.converged)


def test_tolerance_table_matches_reference(small):
    table = small["tol_table"]
    rows = []
    for strat in ("fixed", "dynamic_mid", "dynamic_mid_bl", "dynamic_b",
                  "dynamic_b_bl", "direct_a_iter_b", "iter_a_direct_b"):
        cfg = orc.Config(strategy=strat, gap_budget=3e-7, kmax=40)
        for k in (1, 2, 7):
            for (uu, vv) in ((0.0, 0.0), (1e-10, 3e-11)):
                eh = orc.tolerance_budget(cfg, k, uu, vv)
                for nw, nt in ((1.0, 2.0), (3e-4, 1e-6), (5e-9, 2e-3)):
                    dA, dB, cA, cB = orc.choose_tolerances(cfg, k, nw, nt, eh)
                    rows.append([eh, dA, dB, float(cA), float(cB)])
    assert np.array_equal(np.array(rows), table)


def test_computed_residual_norm_matches_reference(small):
    got = orc.computed_residual_norm(small["crn_w"], small["crn_t"])
    assert abs(got - small["crn"][0]) <= 1e-14 * small["crn"][0]


# -- the ADI driver restatement against the reference's own runs ------------------

def _c1_oracle_run(strategy, solver):
    spec = cfgs.CONFIGS["c1"]
    A, B, M, C, f, g = cfgs.build_problem("c1")
    pairs, cyclic = spec.load_shift_pairs()
    cfg = orc.Config(strategy=strategy, kmax=spec.kmax)
    bA = orc.Binding("A", A, None, solver=solver, restart=spec.restart)
    bB = orc.Binding("B", B, None, solver=solver, restart=spec.restart)
    return orc.run_adi(A, B, f, g, cfg, pairs, bA, bB, cyclic=cyclic)


@pytest.mark.parametrize("strategy", ["dynamic_mid_bl", "fixed"])
def test_oracle_bicgstab_adi_matches_reference_c1(strategy):
    """The restated driver + restated BiCGstab reproduce the reference's
    run_with_state on config 1 step by step (golden from the reference)."""
    gold = read_steps_csv(os.path.join(GOLD, f"ref_c1_{strategy}_bicgstab.csv"))
    run = _c1_oracle_run(strategy, "bicgstab")
    assert run.outer_iterations == len(gold) == 91
    for rec, g in zip(run.records, gold):
        assert rec.inner_it_A == g["inner_it_A"] and rec.inner_it_B == g["inner_it_B"]
        assert abs(rec.scaled_res - g["scaled_res"]) <= 1e-9 * g["scaled_res"]
        assert abs(rec.delta_A - g["delta_A"]) <= 1e-9 * g["delta_A"]


def test_oracle_driver_matches_reference_driver_with_gmres():
    """The reference's run_with_state driving the oracle GMRES (golden) equals
    the oracle's own driver -- the driver restatement is exact."""
    gold = read_steps_csv(os.path.join(GOLD, "refdriver_c1_gmres.csv"))
    mine = read_steps_csv(os.path.join(GOLD, "oracle_c1_gmres.csv"))
    assert len(gold) == len(mine) == 91
    for a, b in zip(gold, mine):
        assert a == b


def test_oracle_bicgstab_adi_matches_reference_generalised():
    """Generalised pencils (A, M), (B, C) of the reduced config 3: the restated
    driver (M z, C^T y, assembled Jacobi) reproduces the reference's run."""
    gold = read_steps_csv(os.path.join(GOLD, "ref_c3s_dynamic_mid_bl_bicgstab.csv"))
    spec = cfgs.CONFIGS["c3s"]
    A, B, M, C, f, g = cfgs.build_problem("c3s")
    pairs, cyclic = spec.load_shift_pairs()
    cfg = orc.Config(strategy="dynamic_mid_bl", kmax=150)
    bA = orc.Binding("A", A, M, solver="bicgstab")
    bB = orc.Binding("B", B, C, solver="bicgstab")
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        run = orc.run_adi(A, B, f, g, cfg, pairs, bA, bB, M=M, C=C, cyclic=cyclic)
    assert run.outer_iterations == len(gold)
    for rec, gd in zip(run.records, gold):
        assert rec.inner_it_A == gd["inner_it_A"] and rec.inner_it_B == gd["inner_it_B"]
        assert abs(rec.scaled_res - gd["scaled_res"]) <= 1e-8 * gd["scaled_res"]


@pytest.mark.parametrize("name", ["c1", "c3s"])
def test_true_residual_norm_matches_reference(name):
    """oracle.true_residual_norm reproduces the reference's own value
    (adi.py:682-726) on factors its driver produced (ref_verify_<name>.npz)."""
    gold = np.load(os.path.join(GOLD, f"ref_verify_{name}.npz"))
    A, B, M, C, f, g = cfgs.build_problem(name)
    got = orc.true_residual_norm(A, B, f, g, gold["Z"], gold["Y"], gold["gdiag"], M=M, C=C)
    want = float(gold["true_residual_norm"])
    assert abs(got - want) <= 1e-9 * want, (got, want)


@pytest.mark.parametrize("name", ["c1", "c3s"])
def test_residual_gap_and_factor_identity_match_reference(name):
    """oracle.residual_gap / verify_factor_identity reproduce the reference's
    values (adi.py:632-679) on the state its driver retained
    (keep_inner_residuals=True; ref_verify_<name>.npz)."""
    gold = np.load(os.path.join(GOLD, f"ref_verify_{name}.npz"))
    A, B, M, C, f, g = cfgs.build_problem(name)
    r = f.shape[1]
    args = (A, B, gold["S_A"], gold["S_B"], gold["Z"], gold["Y"])
    gap = orc.residual_gap(*args, gold["gammas"], r, M=M, C=C)
    want = float(gold["residual_gap"])
    assert abs(gap - want) <= 1e-10 * want, (gap, want)
    hist = [tuple(p) for p in gold["shift_history"]]
    fid = orc.verify_factor_identity(*args, gold["w"], gold["t"], gold["gammas"], hist, r,
                                     M=M, C=C)
    # the identity holds to rounding: both values are at the roundoff level
    assert fid <= 1e-15 and float(gold["factor_identity"]) <= 1e-15, (fid, gold["factor_identity"])
    # a defect the identity does not absorb: dropping S^A leaves ||S^A|| / scale
    # on the A side, the same number in the reference's formula
    S0 = np.zeros_like(gold["S_A"])
    fid0 = orc.verify_factor_identity(A, B, S0, gold["S_B"], gold["Z"], gold["Y"], gold["w"],
                                      gold["t"], gold["gammas"], hist, r, M=M, C=C)
    scale = np.linalg.norm(A.data) * np.linalg.norm(gold["Z"])
    assert abs(fid0 - np.linalg.norm(gold["S_A"]) / scale) <= 1e-6 * fid0


# -- MINRES (krylov.py:187-287), pinned to the reference's own outputs -----------

MINRES_CASES = [("def_jac", None, False, "jacobi"), ("indef_jac", None, False, "jacobi"),
                ("def_none_c", None, False, "none"), ("adj_cap", None, True, "jacobi"),
                ("pencil_jac", "pencil_mass", False, "jacobi")]


@pytest.mark.parametrize("name,mass,adjoint,precond", MINRES_CASES)
def test_oracle_minres_matches_reference(name, mass, adjoint, precond):
    """The restated MINRES reproduces the reference's krylov.minres on the
    fixtures of tests/golden/make_golden_minres.py bit for bit: same iteration
    counts, same solutions."""
    d = np.load(os.path.join(GOLD, "ref_minres.npz"))
    A = sp.csr_matrix(d["lap_A24"])
    M = None if mass is None else sp.csr_matrix(d[mass])
    op = orc.ShiftedOp(A, M, complex(d[name + "_shift"][0]), adjoint=adjoint)
    dinv = orc.jacobi_dinv(op) if precond == "jacobi" else None
    res = orc.minres(op, d[name + "_b"], float(d[name + "_delta"][0]),
                     int(d[name + "_maxit"][0]), dinv)
    assert np.array_equal(res.iterations, d[name + "_iters"])
    assert np.array_equal(res.converged, d[name + "_conv"])
    assert np.max(np.abs(res.solution - d[name + "_x"])) <= 1e-14 * np.max(np.abs(d[name + "_x"]))


def test_oracle_minres_known_answers(rng):
    """test_krylov.py:58-98: identity in <= 1 iteration, diagonal negative
    definite against the dense solve, indefinite 2 x 2 in <= 2 iterations, and
    the reference's own output on the 50 x 50 diagonal case."""
    d = np.load(os.path.join(GOLD, "ref_minres.npz"))
    b = rng.standard_normal((4, 1))
    res = orc.minres(orc.ShiftedOp(sp.eye(4, format="csr"), None, 0.0), b, 1e-12)
    assert res.total_iterations <= 1 and np.max(np.abs(res.solution - b)) < 1e-12
    D = np.diag(-np.arange(1.0, 51.0))
    res = orc.minres(orc.ShiftedOp(sp.csr_matrix(D), None, 0.0), d["kat_diag_b"], 1e-10)
    assert np.array_equal(res.iterations, d["kat_diag_iters"])
    assert np.max(np.abs(res.solution - d["kat_diag_x"])) <= 1e-14
    res = orc.minres(orc.ShiftedOp(sp.csr_matrix(np.diag([-1.0, 1.0])), None, 0.0),
                     np.array([[1.0], [1.0]]), 1e-12)
    assert res.total_iterations <= 2
    assert np.max(np.abs(res.solution[:, 0] - np.array([-1.0, 1.0]))) < 1e-10


def test_oracle_reference_dispatch():
    """Binding(solver="reference") follows SolverBinding.uses_minres
    (adi.py:468-472): MINRES for a symmetric side at a real shift, BiCGstab for
    a complex shift or an unsymmetric side."""
    d = np.load(os.path.join(GOLD, "ref_minres.npz"))
    A = sp.csr_matrix(d["lap_A24"])
    b = orc.Binding("A", A, None, solver="reference")
    assert b.uses_minres(-10.0) and not b.uses_minres(-10.0 + 1j)
    U = A + sp.diags(np.ones(A.shape[0] - 1), 1, format="csr")
    assert not orc.Binding("A", U, None, solver="reference").uses_minres(-10.0)
