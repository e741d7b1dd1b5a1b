"""The CLI adapter: the reference's own front end
(sylvadi.cli, installed in oracle/_ref) with the GPU options and the routes
rebound; host-side checks here, the GPU routes in tests/test_gpu_cli.py."""

import json
import os

import numpy as np
import pytest

pytest.importorskip("sylvadi")

from paper_2312_02891_b200 import cli  # noqa: E402


def write(tmp_path, name, obj):
    p = tmp_path / name
    p.write_text(json.dumps(obj))
    return str(p)


BASE = {"problem": {"dimension": 2, "n0_A": 8, "n0_B": 6, "r": 1, "seed": 0},
        "strategies": ["dynamic_mid_bl"], "output_dir": "out"}


@pytest.mark.parametrize("bad", [
    {k: v for k, v in BASE.items() if k != "problem"},
    {**BASE, "strategies": []},
    {**BASE, "strategies": ["nope"]},
    {**BASE, "strategies": ["exact_direct"]},          # direct solves: not on the GPU path
    {**BASE, "config": {"a_mode": "direct"}},          # mixed: direct A side
    {**BASE, "config": {"bogus": 1}},
    {k: v for k, v in BASE.items() if k != "output_dir"},
    {**BASE, "problem": {"files": {"a": "missing.mtx", "b": "x", "f": "y", "g": "z"}}},
    {**BASE, "shifts": {"file": "missing.json"}},
    {**BASE, "gpu": {"solver": "ilu-gmres"}},           # unknown inner solver
    {**BASE, "gpu": {"driver": "cpu"}},                 # no CPU driver
    {**BASE, "gpu": {"blocks": 4}},                     # unknown gpu key
])
def test_manifest_validation_exit_code(tmp_path, bad):
    """Everything the reference validates exits 2 through the adapter (its own
    RunManifest), and so do the GPU-specific errors -- before any device work."""
    path = write(tmp_path, "m.json", bad)
    assert cli.main(["solve", "--manifest", path]) == cli.EXIT_VALIDATION


def test_gpu_options_merge_and_flags():
    o = cli.gpu_options({"restart": 30, "flexible": True}, {"restart": None, "solver": "bicgstab"})
    assert o["restart"] == 30 and o["flexible"] and o["solver"] == "bicgstab"
    assert o["driver"] == "device"
    o = cli.gpu_options({"restart": 30}, {"restart": 12})
    assert o["restart"] == 12                      # flags win
    with pytest.raises(cli.OptionError):
        cli.gpu_options({"restart": 0}, {})
    with pytest.raises(cli.OptionError):
        cli.gpu_options("x", {})


def test_gen_is_the_reference_command(tmp_path):
    """Subcommands without device work run the reference's code unchanged."""
    spec = write(tmp_path, "spec.json", {"dimension": 2, "n0_A": 5, "n0_B": 4, "r": 2,
                                         "seed": 3})
    out = str(tmp_path / "gen")
    assert cli.main(["gen", "--spec", spec, "--out", out]) == cli.EXIT_OK
    from sylvadi.sparse import read_dense_array, read_matrix_market
    A = read_matrix_market(os.path.join(out, "A.mtx"))
    f = read_dense_array(os.path.join(out, "f.mtx"))
    assert A.nrows == 25 and f.shape == (25, 2)


def test_routes_are_restored():
    refcli = cli.reference_cli()
    before = refcli.run_with_state
    with cli.routed(refcli, cli.gpu_options(None, {})):
        assert refcli.run_with_state is not before
    assert refcli.run_with_state is before


def test_results_convert_to_reference_types(tmp_path):
    """The device driver's results become the reference's types, whose own
    writers and readers then apply (report CSV, factor files)."""
    import sylvadi.adi as refadi
    from paper_2312_02891_b200 import adi as gadi
    rng = np.random.default_rng(0)
    Z = rng.standard_normal((7, 4)) + 1j * rng.standard_normal((7, 4))
    Y = rng.standard_normal((5, 4)) + 1j * rng.standard_normal((5, 4))
    sol = gadi.LowRankSolution(Z=Z, gammas=[1 + 2j, -3.0], Y=Y, r=2)
    rep = gadi.SolveReport(rhs_norm=2.0, strategy=gadi.Strategy.DYNAMIC_MID_BL)
    rep.records.append(gadi.StepRecord(1, 0.5, 1e-3, 1e-3, 1e-4, 2e-4, 7, 8, 0.1, 0.2, 1.5))
    rep.outer_iterations, rep.converged, rep.final_scaled_residual = 1, False, 0.5
    st = gadi.AdiState(2, Z, Y, [1 + 2j, -3.0], Z[:, :2], Y[:, :2], 0.1, 0.2,
                       [(-1.0, -2.0), (-3.0, -4.0)], [], [], False)
    rsol, rrep, rst = cli._to_reference_results(refadi, sol, rep, st, 2)
    assert isinstance(rsol, refadi.LowRankSolution) and isinstance(rrep, refadi.SolveReport)
    rrep.to_csv(str(tmp_path / "report.csv"))
    rows = (tmp_path / "report.csv").read_text().splitlines()
    assert rows[0] == refadi.CSV_HEADER and rows[1].startswith("1,5.0")
    rsol.save(str(tmp_path))
    back = refadi.LowRankSolution.load(str(tmp_path), r=2)
    assert np.array_equal(back.Z, Z) and np.array_equal(back.gamma_diag(), sol.gamma_diag())
    assert rst.k == 2 and rst.shift_history[1] == (-3.0, -4.0)
