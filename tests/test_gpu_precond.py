"""The reference's incomplete-factorisation preconditioners on the device
(sad_pc_create / sad_pc_apply / sad_bicg_solve_pc /
sad_minres_solve_pc) against the REFERENCE's own factors, actions, solves and
ADI records (tests/golden/ref_precond.npz, ref_c1_*_bicgstab.csv,
ref_sym_ict_minres.csv; written by tests/golden/make_golden_precond.py from
precond.py / krylov.py / adi.py) and against the oracle restatement."""

import json
import os
import warnings

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import precond as opc
from oracle import sylvadi_oracle as orc

from conftest import GOLD, read_steps_csv
from precond_cases import CASES, Case

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _device_precond(case):
    from paper_2312_02891_b200.device import DeviceMatrix, DevicePrecond
    base = DeviceMatrix(case.base, case.adjoint, 0)
    mass = None if case.mass is None else DeviceMatrix(case.mass, case.adjoint, 0)
    return DevicePrecond(base, mass, case.shift, case.adjoint, case.kind, case.droptol)


@pytest.mark.parametrize("name", CASES)
def test_factors_bit_identical_to_reference(name):
    """factorize (precond.py:307-357): L, U / G are the reference's, bit for bit."""
    case = Case(name)
    pc = _device_precond(case)
    if case.lu is not None:
        li, lj, lv = pc.factor(0)
        ui, uj, uv = pc.factor(1)
        for got, ref in zip((li, lj, lv, ui, uj, uv), case.lu):
            assert got.shape == ref.shape
            assert np.array_equal(got, ref)
        assert not pc.is_spd_capable
    else:
        for got, ref in zip(pc.factor(0), case.chol):
            assert got.shape == ref.shape
            assert np.array_equal(got, ref)
        assert pc.sign == case.sign and pc.is_spd_capable
    assert pc.is_complex == (case.shift.imag != 0.0)
    assert pc.levels[0] >= 1 and pc.levels[1] >= 1


@pytest.mark.parametrize("name", CASES)
def test_apply_bit_identical_to_reference(name):
    """apply / apply_spd (precond.py:224-256): the level-scheduled device solves
    subtract in the reference's order with single roundings -> identical bits,
    for complex blocks of every width and (real factors) real blocks."""
    case = Case(name)
    pc = _device_precond(case)
    x = torch.from_numpy(case.x).cuda()
    got = pc.apply(x).cpu().numpy()
    assert np.array_equal(got, case.apply)
    # in place, and again (epoch flags are reused without clearing)
    y = x.clone()
    pc.apply(y, y)
    assert np.array_equal(y.cpu().numpy(), case.apply)
    if case.apply_spd is not None:
        assert np.array_equal(pc.apply(x, spd=True).cpu().numpy(), case.apply_spd)
    else:
        with pytest.raises(ValueError):
            pc.apply(x, spd=True)
    # other block widths against the oracle (columns are independent)
    op = orc.ShiftedOp(case.base, case.mass, case.shift, adjoint=case.adjoint)
    fact = opc.factorize(opc.assembled(op), case.kind, case.droptol)
    rng = np.random.default_rng(3)
    for r in (1, 5, 8):
        xb = rng.standard_normal((pc.n, r)) + 1j * rng.standard_normal((pc.n, r))
        got = pc.apply(torch.from_numpy(xb).cuda()).cpu().numpy()
        assert np.array_equal(got, fact.apply(xb))
    xr = rng.standard_normal((pc.n, 3))
    if pc.is_complex:
        with pytest.raises(ValueError):
            pc.apply(torch.from_numpy(xr).cuda())
    else:
        got = pc.apply(torch.from_numpy(xr).cuda()).cpu().numpy()
        assert np.array_equal(got, fact.apply(xr).real)


def test_breakdowns_raise_like_the_reference():
    """precond.py:89-92 / 285-286 -> FactorizationBreakdown; the binding falls
    back to Jacobi with a warning (adi.py:458-465)."""
    from paper_2312_02891_b200 import GpuGmresBinding, _lib
    from paper_2312_02891_b200.device import DeviceMatrix, DevicePrecond
    z = sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]]))
    with pytest.raises(_lib.FactorizationBreakdown, match="zero pivot in ilu0"):
        DevicePrecond(DeviceMatrix(z, False, 0), None, 0.0, False, "ilu0", 0.0)
    lap = Case("lap16_ic0_0").base
    with pytest.raises(_lib.FactorizationBreakdown, match="not positive definite"):
        DevicePrecond(DeviceMatrix(lap, False, 0), None, 500.0, False, "ic0", 0.0)
    gb = GpuGmresBinding("A", lap, None, precond_kind="ic0", solver="reference")
    with pytest.warns(UserWarning, match="falling back to Jacobi"):
        op = gb.operator(500.0)
    assert op.pc is None and op.precond_kind == "jacobi"
    with pytest.raises(ValueError):
        GpuGmresBinding("A", lap, None, precond_kind="ilut", solver="gmres")
    with pytest.raises(ValueError):
        GpuGmresBinding("A", lap, None, precond_kind="ilu7", solver="reference")


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("solver", ["bicgstab", "minres"])
def test_preconditioned_solves_match_reference(name, solver):
    """bicgstab / minres(InnerSolveRequest(..., preconditioner=fact))
    (krylov.py:160-184, 271-287): MINRES counts within +-2 of the reference's,
    BiCGstab within the band its counts move in under rounding noise (+-3, see
    tests/test_gpu_bicgstab.py), same flags, solutions to the solve tolerance."""
    from paper_2312_02891_b200 import GpuGmresBinding
    case = Case(name)
    ref = case.solve(solver)
    if ref is None:
        pytest.skip("solver not recorded for this case")
    gb = GpuGmresBinding(case.side, case.base, case.mass, precond_kind=case.kind,
                         droptol=case.droptol, solver=solver)
    delta = float(ref["delta"][0])
    got = gb.solve(case.shift, ref["b"], delta)
    band = 2 if solver == "minres" else 3
    assert np.all(np.abs(got.iterations - ref["iters"]) <= band), (got.iterations, ref["iters"])
    assert np.array_equal(got.converged, ref["conv"])
    assert np.all(got.achieved_residual_norms <= delta / ref["b"].shape[1])
    assert np.linalg.norm(got.solution - ref["x"]) <= 1e-6 * np.linalg.norm(ref["x"])
    op = orc.ShiftedOp(case.base, case.mass, case.shift, adjoint=case.adjoint)
    true = ref["b"] - op.apply(got.solution)
    assert np.max(np.abs(true - got.residual)) <= 1e-9 * np.max(np.abs(ref["b"]))


def test_reference_dispatch_with_cholesky_kinds():
    """adi.py:468-472: a symmetric side at a real shift with ic0/ict runs MINRES,
    a complex shift or an ILU kind BiCGstab."""
    from paper_2312_02891_b200 import GpuGmresBinding
    lap = Case("lap16_ic0_0").base
    gb = GpuGmresBinding("A", lap, None, precond_kind="ict", droptol=0.1, solver="reference")
    assert gb.kind_for(-10.0) == "minres" and gb.kind_for(-10.0 + 1j) == "bicgstab"
    gb = GpuGmresBinding("A", lap, None, precond_kind="ilut", droptol=0.1, solver="reference")
    assert gb.kind_for(-10.0) == "bicgstab"


def _device_adi(A, B, f, g, pairs, cyclic, kind, kmax):
    import paper_2312_02891_b200 as pb
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
    cfg = pb.AdiConfig(strategy="dynamic_mid_bl", kmax=kmax, precond_kind_A=kind,
                       precond_kind_B=kind, precond_droptol_A=0.1, precond_droptol_B=0.1)
    eng = pb.DeviceAdi(prob, cfg, pb.ShiftSequence(pairs=pairs, cyclic=cyclic), solver="reference")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return eng.run()


@pytest.mark.parametrize("kind", ["ilut", "ilu0"])
def test_c1_adi_with_ilu_matches_reference_records(kind):
    """Config 1 through the device driver with the paper's preconditioner and the
    reference's own solver dispatch, against the reference's run_with_state
    records: same outer steps, scaled residual history, inner counts within
    max(2, 10 %) per step (BiCGstab's noise band) and 3 % in total."""
    from paper_2312_02891_b200 import configs as cfgs
    A, B, M, C, f, g = cfgs.build_problem("c1")
    pairs, cyclic = cfgs.CONFIGS["c1"].load_shift_pairs()
    sol, rep, _ = _device_adi(A, B, f, g, pairs, cyclic, kind, 150)
    ref = read_steps_csv(os.path.join(GOLD, f"ref_c1_{kind}_bicgstab.csv"))
    assert rep.converged and rep.outer_iterations == len(ref)
    for got, want in zip(rep.records, ref):
        assert abs(got.scaled_res - want["scaled_res"]) <= 1e-6 * want["scaled_res"]
        for side in ("A", "B"):
            gi, wi = getattr(got, f"inner_it_{side}"), want[f"inner_it_{side}"]
            assert abs(gi - wi) <= max(2, 0.1 * wi), (got.step, side, gi, wi)
    tot_ref = sum(w["inner_it_A"] + w["inner_it_B"] for w in ref)
    assert abs(rep.sum_inner_A + rep.sum_inner_B - tot_ref) <= 0.03 * tot_ref


def test_symmetric_adi_with_ict_minres_matches_reference_records():
    """Symmetric Laplacian pair, ICT(0.1) on both sides: every inner solve is
    split-preconditioned MINRES (adi.py:468-488); records of the reference's
    run_with_state, inner counts +-2 per step."""
    from paper_2312_02891_b200.problems import convdiff_fd, random_rhs
    with open(os.path.join(GOLD, "ref_sym_shifts.json")) as fh:
        meta = json.load(fh)
    A = convdiff_fd(2, meta["n0_A"])
    B = convdiff_fd(2, meta["n0_B"])
    f, g = random_rhs(A.shape[0], B.shape[0], meta["r"], meta["seed"])
    pairs = [tuple(p) for p in meta["pairs"]]
    sol, rep, _ = _device_adi(A, B, f, g, pairs, True, "ict", meta["kmax"])
    ref = read_steps_csv(os.path.join(GOLD, "ref_sym_ict_minres.csv"))
    assert rep.converged and rep.outer_iterations == len(ref)
    for got, want in zip(rep.records, ref):
        assert abs(got.scaled_res - want["scaled_res"]) <= 1e-6 * want["scaled_res"]
        assert abs(got.inner_it_A - want["inner_it_A"]) <= 2
        assert abs(got.inner_it_B - want["inner_it_B"]) <= 2
