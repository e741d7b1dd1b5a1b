"""Pin the oracle's incomplete factorisations (oracle/precond.py +
oracle/precond_oracle.c) to the REFERENCE's own factors, actions and
preconditioned solves (tests/golden/ref_precond.npz, written by running
/root/reference/pkg/src/sylvadi/precond.py in the build container).  CPU only.
"""

import os
import warnings

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import precond as opc
from oracle import sylvadi_oracle as orc
from paper_2312_02891_b200 import configs as cfgs

from conftest import GOLD, read_steps_csv
from precond_cases import CASES, Case, data


def _factor(case):
    op = orc.ShiftedOp(case.base, case.mass, case.shift, adjoint=case.adjoint)
    return op, opc.factorize(opc.assembled(op), case.kind, case.droptol)


@pytest.mark.parametrize("name", CASES)
def test_factors_bit_identical_to_reference(name):
    # precond.py:34-125, 279-304, 307-357
    case = Case(name)
    _, fact = _factor(case)
    if case.lu is not None:
        for got, ref in zip(fact.lu, case.lu):
            assert got.shape == ref.shape
            assert np.array_equal(got, ref)
    else:
        assert fact.sign == case.sign
        for got, ref in zip(fact.chol, case.chol):
            assert got.shape == ref.shape
            assert np.array_equal(got, ref)


@pytest.mark.parametrize("name", CASES)
def test_apply_bit_identical_to_reference(name):
    # precond.py:129-173, 224-256
    case = Case(name)
    _, fact = _factor(case)
    assert np.array_equal(fact.apply(case.x), case.apply)
    if case.apply_spd is not None:
        assert np.array_equal(fact.apply_spd(case.x), case.apply_spd)
    # one column, 1-D in / 1-D out
    assert np.array_equal(fact.apply(case.x[:, 0]), case.apply[:, 0])


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("solver", ["bicgstab", "minres"])
def test_preconditioned_solves_match_reference(name, solver):
    # krylov.py:160-184 / 271-287 with preconditioner=IncompleteFactorization
    case = Case(name)
    ref = case.solve(solver)
    if ref is None:
        pytest.skip("solver not recorded for this case")
    op, fact = _factor(case)
    fn = orc.minres if solver == "minres" else orc.bicgstab
    got = fn(op, ref["b"], float(ref["delta"][0]), 1000, fact)
    assert np.array_equal(got.iterations, ref["iters"])
    assert np.array_equal(got.converged, ref["conv"])
    assert np.linalg.norm(got.solution - ref["x"]) <= 1e-12 * np.linalg.norm(ref["x"])


def test_breakdowns():
    # precond.py:89-92 (zero pivot), 285-286 (indefinite for the Cholesky kinds)
    d = data()
    z = sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]]))
    with pytest.raises(opc.FactorizationBreakdown) as e:
        opc.factorize(z, "ilu0")
    assert str(e.value) == str(d["break_zero_pivot_msg"][0])
    lap = Case("lap16_ic0_0").base
    with pytest.raises(opc.FactorizationBreakdown) as e:
        opc.factorize(lap + 500.0 * sp.eye(256, format="csr"), "ic0")
    assert str(e.value) == str(d["break_indef_msg"][0])
    with pytest.raises(ValueError):
        opc.factorize(lap, "ilu7")
    # precond.py:244-245
    _, fact = _factor(Case("cd12_ilu0_0"))
    with pytest.raises(ValueError):
        fact.apply_spd(np.ones(144))


@pytest.mark.parametrize("kind", ["ilut", "ilu0"])
def test_oracle_adi_with_ilu_matches_reference_c1(kind):
    """The reference's run_with_state on config 1 with its own ILU-BiCGstab path
    (adi.py:553-607, 453-466), step for step."""
    A, B, M, C, f, g = cfgs.build_problem("c1")
    spec = cfgs.CONFIGS["c1"]
    pairs, cyclic = spec.load_shift_pairs()
    cfg = orc.Config(strategy="dynamic_mid_bl", kmax=150)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        run = orc.run_adi(A, B, f, g, cfg, pairs,
                          orc.Binding("A", A, None, solver="reference", precond=kind, droptol=0.1),
                          orc.Binding("B", B, None, solver="reference", precond=kind, droptol=0.1),
                          cyclic=cyclic)
    ref = read_steps_csv(os.path.join(GOLD, f"ref_c1_{kind}_bicgstab.csv"))
    assert len(run.records) == len(ref)
    for got, want in zip(run.records, ref):
        assert got.inner_it_A == want["inner_it_A"] and got.inner_it_B == want["inner_it_B"]
        assert abs(got.scaled_res - want["scaled_res"]) <= 1e-9 * want["scaled_res"]
        assert abs(got.delta_A - want["delta_A"]) <= 1e-9 * want["delta_A"]
