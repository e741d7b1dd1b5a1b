"""The reference's inner solver for Hermitian sides on the device
(sad_minres_solve): split-preconditioned MINRES (krylov.py:187-287), against
the reference's own outputs (tests/golden/ref_minres.npz, written by
tests/golden/make_golden_minres.py from krylov.minres) and, at the ADI level,
against the reference's run_with_state on a symmetric pair, where its
SolverBinding sends every inner solve to MINRES (adi.py:468-488)."""

import json
import os
import warnings

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import sylvadi_oracle as orc

from conftest import GOLD, read_steps_csv

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CASES = [("def_jac", None, "A", "jacobi"), ("indef_jac", None, "A", "jacobi"),
         ("def_none_c", None, "A", "none"), ("adj_cap", None, "B", "jacobi"),
         ("pencil_jac", "pencil_mass", "A", "jacobi")]


def _gold():
    return np.load(os.path.join(GOLD, "ref_minres.npz"))


@pytest.mark.parametrize("name,mass,side,precond", CASES)
@pytest.mark.parametrize("solver", ["minres", "reference"])
def test_minres_matches_reference(name, mass, side, precond, solver):
    """Same iteration counts as the reference's krylov.minres (+-2; the
    device reductions sum in a different order), same convergence flags,
    solutions within the solve tolerance, the true residual returned."""
    from paper_2312_02891_b200 import GpuGmresBinding
    d = _gold()
    A = sp.csr_matrix(d["lap_A24"])
    M = None if mass is None else sp.csr_matrix(d[mass])
    shift = complex(d[name + "_shift"][0])
    b = d[name + "_b"]
    delta = float(d[name + "_delta"][0])
    maxit = int(d[name + "_maxit"][0])
    gb = GpuGmresBinding(side, A, M, precond_kind=precond, max_iterations=maxit, solver=solver)
    assert gb.kind_for(shift) == "minres"
    got = gb.solve(shift, b, delta)
    want_it = d[name + "_iters"]
    assert np.all(np.abs(got.iterations - want_it) <= 2), (got.iterations, want_it)
    assert np.array_equal(got.converged, d[name + "_conv"])
    if np.all(d[name + "_conv"]):
        assert np.all(got.achieved_residual_norms <= delta / b.shape[1])
        x = d[name + "_x"]
        assert np.linalg.norm(got.solution - x) <= 1e-6 * np.linalg.norm(x)
    op = orc.ShiftedOp(A, M, shift, adjoint=(side == "B"))
    true = b - op.apply(got.solution)
    assert np.max(np.abs(true - got.residual)) <= 1e-9 * np.max(np.abs(b))


def test_minres_known_answers(rng):
    """test_krylov.py:58-98 through the device: identity in <= 1 iteration,
    negative definite diagonal against the dense solve (and the reference's
    own count), indefinite 2 x 2 in <= 2, zero column -> 0 iterations, the
    per-column bound delta / r."""
    from paper_2312_02891_b200 import GpuGmresBinding
    d = _gold()

    def run(dense, b, delta, maxit=1000):
        gb = GpuGmresBinding("A", sp.csr_matrix(dense), None, precond_kind="none",
                             max_iterations=maxit, solver="minres")
        return gb.solve(0.0, b, delta)

    b = rng.standard_normal((4, 1))
    res = run(np.eye(4), b, 1e-12)
    assert res.iterations.sum() <= 1 and np.max(np.abs(res.solution - b)) < 1e-12
    D = np.diag(-np.arange(1.0, 51.0))
    res = run(D, d["kat_diag_b"], 1e-10)
    assert abs(int(res.iterations[0]) - int(d["kat_diag_iters"][0])) <= 2
    assert np.max(np.abs(res.solution - np.linalg.solve(D, d["kat_diag_b"]))) < 1e-8
    res = run(np.diag([-1.0, 1.0]), np.array([[1.0], [1.0]]), 1e-12)
    assert res.iterations.sum() <= 2
    assert np.max(np.abs(res.solution[:, 0] - np.array([-1.0, 1.0]))) < 1e-10
    D = np.diag(-np.arange(1.0, 21.0))
    bb = rng.standard_normal((20, 4))
    bb[:, 2] = 0.0
    res = run(D, bb, 1e-9)
    assert np.all(res.converged) and res.iterations[2] == 0
    assert np.all(res.solution[:, 2] == 0)
    assert np.all(res.achieved_residual_norms <= 1e-9 / 4)


def test_minres_dispatch_and_errors(rng):
    """solver="reference" follows uses_minres (adi.py:468-472); MINRES at a
    complex shift is an error, not a silent fallback."""
    from paper_2312_02891_b200 import GpuGmresBinding
    d = _gold()
    A = sp.csr_matrix(d["lap_A24"])
    gb = GpuGmresBinding("A", A, None, solver="reference")
    assert gb.kind_for(-10.0) == "minres" and gb.kind_for(-10.0 + 2.0j) == "bicgstab"
    U = A + sp.diags(np.ones(A.shape[0] - 1), 1, format="csr")
    assert GpuGmresBinding("A", U, None, solver="reference").kind_for(-10.0) == "bicgstab"
    # a complex shift through the reference dispatch runs BiCGstab and converges
    b = rng.standard_normal((A.shape[0], 1))
    res = gb.solve(-10.0 + 2.0j, b, 1e-8)
    assert np.all(res.converged)
    gm = GpuGmresBinding("A", A, None, solver="minres")
    with pytest.raises(ValueError):
        gm.solve(-10.0 + 2.0j, b.astype(complex), 1e-8)


def test_minres_adi_symmetric_matches_reference():
    """The device ADI with the reference's own inner-solver dispatch (every
    solve MINRES here) against the reference's run_with_state records: same
    outer steps, scaled residual history to 1e-6, per-step inner counts
    within +-2 and the totals within 1 %."""
    import paper_2312_02891_b200 as pb
    from paper_2312_02891_b200.problems import convdiff_fd, random_rhs
    meta = json.load(open(os.path.join(GOLD, "ref_sym_shifts.json")))
    A = convdiff_fd(2, meta["n0_A"])
    B = convdiff_fd(2, meta["n0_B"])
    f, g = random_rhs(A.shape[0], B.shape[0], meta["r"], meta["seed"])
    pairs = [tuple(p) for p in meta["pairs"]]
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
    cfg = pb.AdiConfig(strategy="dynamic_mid_bl", kmax=meta["kmax"],
                       precond_kind_A="jacobi", precond_kind_B="jacobi")
    seq = pb.ShiftSequence(pairs=pairs, cyclic=True)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        sol, rep, _ = pb.run_with_state(prob, cfg, seq, solver="reference")
    gold = read_steps_csv(os.path.join(GOLD, "ref_sym_dynamic_mid_bl_minres.csv"))
    assert rep.converged
    assert rep.outer_iterations == len(gold)
    for rec, gd in zip(rep.records, gold):
        for got, want in ((rec.inner_it_A, gd["inner_it_A"]), (rec.inner_it_B, gd["inner_it_B"])):
            assert abs(got - want) <= 2, (rec.step, got, want)
        assert abs(rec.scaled_res - gd["scaled_res"]) <= 1e-6 * gd["scaled_res"]
    for key, tot in (("inner_it_A", rep.sum_inner_A), ("inner_it_B", rep.sum_inner_B)):
        ref = sum(gd[key] for gd in gold)
        assert abs(tot - ref) <= 0.01 * ref
