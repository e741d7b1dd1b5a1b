"""The CLI's GPU routes end to end: solve (device shifts, device ADI, device
true residual) then verify on the stored factors."""

import json
import os

import pytest

from paper_2312_02891_b200 import cli

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def test_solve_then_verify(tmp_path):
    man = {"problem": {"dimension": 2, "n0_A": 16, "n0_B": 12, "r": 2, "seed": 1,
                       "omega_A": [10.0, 10.0], "omega_B": [5.0, -5.0]},
           "strategies": ["fixed", "dynamic_mid_bl"], "shifts": {"pairs": 6},
           "config": {"kmax": 100}, "output_dir": "run", "save_factors": True,
           "gpu": {"restart": 20}}
    path = tmp_path / "m.json"
    path.write_text(json.dumps(man))
    assert cli.main(["solve", "--manifest", str(path)]) == cli.EXIT_OK
    out = tmp_path / "run"
    summ = json.loads((out / "summary.json").read_text())
    for name in ("fixed", "dynamic_mid_bl"):
        e = summ["strategies"][name]
        assert e["converged"] and e["scaled_true_residual"] < 2e-8
        assert (out / name / "report.csv").exists() and (out / name / "Z.mtx").exists()
    assert summ["strategies"]["dynamic_mid_bl"]["savings_vs_fixed"] is not None
    assert os.path.exists(out / "shifts.json") and os.path.exists(out / "problem" / "A.mtx")
    assert cli.main(["verify", "--dir", str(out)]) == cli.EXIT_OK
    ver = json.loads((out / "verify.json").read_text())
    for name in ("fixed", "dynamic_mid_bl"):
        assert abs(ver[name]["scaled_true_residual"]
                   - summ["strategies"][name]["scaled_true_residual"]) < 1e-12


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
    a symmetric pair (omega = 0: MINRES on the device at every real shift,
    BiCGstab otherwise) converges to the outer tolerance through the CLI."""
    man = {"problem": {"dimension": 2, "n0_A": 16, "n0_B": 12, "r": 1, "seed": 2},
           "strategies": ["dynamic_mid_bl"], "shifts": {"pairs": 6},
           "config": {"kmax": 100, "precond_kind_A": "jacobi", "precond_kind_B": "jacobi"},
           "output_dir": "run", "gpu": {"solver": "reference"}}
    path = tmp_path / "m.json"
    path.write_text(json.dumps(man))
    assert cli.main(["solve", "--manifest", str(path)]) == cli.EXIT_OK
    summ = json.loads((tmp_path / "run" / "summary.json").read_text())
    assert summ["inner_solver"] == "gpu reference"
    e = summ["strategies"]["dynamic_mid_bl"]
    assert e["converged"] and e["scaled_true_residual"] < 2e-8
