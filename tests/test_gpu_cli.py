"""The GPU routes of the reference's own front end and the
drop-in proof: the reference's run_with_state driving GpuGmresBinding."""

import json
import os
import warnings

import numpy as np
import pytest

from conftest import GOLD, read_steps_csv

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
sv = pytest.importorskip("sylvadi")          # the reference (oracle/_ref)

from paper_2312_02891_b200 import cli  # noqa: E402
from paper_2312_02891_b200 import configs as cfgs  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def test_reference_driver_with_gpu_bindings_matches_golden():
    """The unchanged reference driver (adi.py:553-607) with GpuGmresBinding on
    both sides (its bindings= seam, adi.py:513-516) reproduces the per-step
    records of the same driver with the oracle's GMRES binding
    (refdriver_c1_gmres.csv): same outer steps, inner counts within +-2."""
    from paper_2312_02891_b200 import GpuGmresBinding
    A, B, M, C, f, g = cfgs.build_problem("c1")
    problem = sv.SylvesterProblem(A=sv.SparseMatrix(A), B=sv.SparseMatrix(B), f=f, g=g)
    seq = sv.ShiftSequence.from_json(cfgs.CONFIGS["c1"].shift_file)
    cfg = sv.AdiConfig(strategy="dynamic_mid_bl", kmax=150)
    bind = sv.adi.SolverBindings(A=GpuGmresBinding("A", problem.A, None, restart=50),
                                 B=GpuGmresBinding("B", problem.B, None, restart=50))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        sol, rep, _ = sv.run_with_state(problem, cfg, seq, bindings=bind)
    gold = read_steps_csv(os.path.join(GOLD, "refdriver_c1_gmres.csv"))
    assert rep.outer_iterations == len(gold) and rep.converged
    for rec, gd in zip(rep.records, gold):
        assert abs(rec.inner_it_A - gd["inner_it_A"]) <= 2, (rec.step, rec.inner_it_A, gd)
        assert abs(rec.inner_it_B - gd["inner_it_B"]) <= 2, (rec.step, rec.inner_it_B, gd)
        assert abs(rec.scaled_res - gd["scaled_res"]) <= 1e-6 * gd["scaled_res"] + 1e-14
    assert isinstance(sol, sv.LowRankSolution)


@pytest.mark.parametrize("driver", ["device", "bindings"])
def test_solve_then_verify(tmp_path, driver):
    man = {"problem": {"dimension": 2, "n0_A": 16, "n0_B": 12, "r": 2, "seed": 1,
                       "omega_A": [10.0, 10.0], "omega_B": [5.0, -5.0]},
           "strategies": ["fixed", "dynamic_mid_bl"], "shifts": {"pairs": 6},
           "config": {"kmax": 100, "keep_inner_residuals": True}, "output_dir": "run",
           "save_factors": True, "gpu": {"restart": 20, "driver": driver}}
    path = tmp_path / "m.json"
    path.write_text(json.dumps(man))
    assert cli.main(["solve", "--manifest", str(path)]) == cli.EXIT_OK
    out = tmp_path / "run"
    summ = json.loads((out / "summary.json").read_text())
    assert summ["gpu"]["driver"] == driver and summ["gpu"]["restart"] == 20
    for name in ("fixed", "dynamic_mid_bl"):
        e = summ["strategies"][name]
        assert e["converged"] and e["scaled_true_residual"] < 2e-8
        assert (out / name / "report.csv").exists() and (out / name / "Z.mtx").exists()
        assert (out / name / "diagnostics" / "S_A.mtx").exists()
    assert summ["strategies"]["dynamic_mid_bl"]["savings_vs_fixed"] is not None
    assert os.path.exists(out / "shifts.json") and os.path.exists(out / "problem" / "A.mtx")
    assert cli.main(["verify", "--dir", str(out)]) == cli.EXIT_OK
    ver = json.loads((out / "verify.json").read_text())
    for name in ("fixed", "dynamic_mid_bl"):
        v = ver[name]
        # the reference's verify keys (cli.py:335-345), computed on the device
        assert set(v) == {"scaled_true_residual", "residual_gap", "gap_estimate_u_plus_v",
                          "gap_bounded_by_estimate", "factor_identity_defect"}
        assert abs(v["scaled_true_residual"] - summ["strategies"][name]["scaled_true_residual"]) < 1e-12
        assert v["gap_bounded_by_estimate"] and v["factor_identity_defect"] < 1e-12


def test_shifts_subcommand(tmp_path):
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps({"dimension": 2, "n0_A": 10, "n0_B": 8, "r": 1}))
    gen = tmp_path / "gen"
    assert cli.main(["gen", "--spec", str(spec), "--out", str(gen)]) == cli.EXIT_OK
    out = tmp_path / "shifts.json"
    assert cli.main(["shifts", "--a", str(gen / "A.mtx"), "--b", str(gen / "B.mtx"),
                     "--pairs", "4", "--out", str(out)]) == cli.EXIT_OK
    assert len(json.loads(out.read_text())["pairs"]) == 4


def test_solve_reference_dispatch_symmetric(tmp_path):
    """gpu.solver = "reference": the reference's own inner-solver dispatch on
    a symmetric pair (MINRES on the device at every real shift, BiCGstab
    otherwise) converges to the outer tolerance through the CLI."""
    man = {"problem": {"dimension": 2, "n0_A": 16, "n0_B": 12, "r": 1, "seed": 2},
           "strategies": ["dynamic_mid_bl"], "shifts": {"pairs": 6},
           "config": {"kmax": 100, "precond_kind_A": "jacobi", "precond_kind_B": "jacobi"},
           "output_dir": "run"}
    path = tmp_path / "m.json"
    path.write_text(json.dumps(man))
    assert cli.main(["--solver", "reference", "solve", "--manifest", str(path)]) == cli.EXIT_OK
    summ = json.loads((tmp_path / "run" / "summary.json").read_text())
    assert summ["gpu"]["solver"] == "reference"
    e = summ["strategies"]["dynamic_mid_bl"]
    assert e["converged"] and e["scaled_true_residual"] < 2e-8


def test_reference_driver_with_gpu_ilut_bindings_matches_reference_records():
    """The unchanged reference driver with the GPU binding carrying the PAPER's
    preconditioner (ILUT(0.1), the reference's own solver dispatch on the
    device): the per-step records of the reference's own ILUT-BiCGstab run on
    config 1 (ref_c1_ilut_bicgstab.csv) -- same outer steps, residual history,
    inner counts within BiCGstab's noise band."""
    from paper_2312_02891_b200 import GpuGmresBinding
    A, B, M, C, f, g = cfgs.build_problem("c1")
    problem = sv.SylvesterProblem(A=sv.SparseMatrix(A), B=sv.SparseMatrix(B), f=f, g=g)
    seq = sv.ShiftSequence.from_json(cfgs.CONFIGS["c1"].shift_file)
    cfg = sv.AdiConfig(strategy="dynamic_mid_bl", kmax=150, precond_kind_A="ilut",
                       precond_kind_B="ilut", precond_droptol_A=0.1, precond_droptol_B=0.1)
    bind = sv.adi.SolverBindings(
        A=GpuGmresBinding("A", problem.A, None, "iterative", "ilut", 0.1, solver="reference"),
        B=GpuGmresBinding("B", problem.B, None, "iterative", "ilut", 0.1, solver="reference"))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        sol, rep, _ = sv.run_with_state(problem, cfg, seq, bindings=bind)
    gold = read_steps_csv(os.path.join(GOLD, "ref_c1_ilut_bicgstab.csv"))
    assert rep.outer_iterations == len(gold) and rep.converged
    for rec, gd in zip(rep.records, gold):
        assert abs(rec.scaled_res - gd["scaled_res"]) <= 1e-6 * gd["scaled_res"] + 1e-14
        for side in ("A", "B"):
            got, want = getattr(rec, f"inner_it_{side}"), gd[f"inner_it_{side}"]
            assert abs(got - want) <= max(2, 0.1 * want), (rec.step, side, got, want)


def test_solve_with_the_papers_preconditioner_through_the_cli(tmp_path):
    """Manifest config precond_kind_* = ilut / droptol 0.1 (the reference's manifest keys,
    cli.py:29-34) with gpu.solver = "reference": factorisation per shift, device
    triangular solves inside BiCGstab, converged run, verify passes."""
    man = {"problem": {"dimension": 2, "n0_A": 16, "n0_B": 12, "r": 2, "seed": 1,
                       "omega_A": [10.0, 10.0], "omega_B": [5.0, -5.0]},
           "strategies": ["dynamic_mid_bl"], "shifts": {"pairs": 6},
           "config": {"kmax": 100, "precond_kind_A": "ilut", "precond_droptol_A": 0.1,
                      "precond_kind_B": "ilu0"},
           "output_dir": "run", "save_factors": True, "gpu": {"solver": "reference"}}
    path = tmp_path / "m.json"
    path.write_text(json.dumps(man))
    assert cli.main(["solve", "--manifest", str(path)]) == cli.EXIT_OK
    out = tmp_path / "run"
    e = json.loads((out / "summary.json").read_text())["strategies"]["dynamic_mid_bl"]
    assert e["converged"] and e["scaled_true_residual"] < 2e-8
    assert cli.main(["verify", "--dir", str(out)]) == cli.EXIT_OK
