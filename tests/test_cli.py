"""CLI front end: manifest validation, problem/factor files
and exit codes as the reference's cli.py; the GPU routes are in
tests/test_gpu_cli.py."""

import json
import os

import numpy as np
import pytest

from paper_2312_02891_b200 import cli


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
    {**BASE, "config": {"bogus": 1}},
    {k: v for k, v in BASE.items() if k != "output_dir"},
    {**BASE, "problem": {"files": {"a": "missing.mtx", "b": "x", "f": "y", "g": "z"}}},
    {**BASE, "shifts": {"file": "missing.json"}},
    {**BASE, "gpu": {"solver": "ilu-gmres"}},           # unknown inner solver
])
def test_manifest_validation_exit_code(tmp_path, bad):
    path = write(tmp_path, "m.json", bad)
    assert cli.main(["solve", "--manifest", path]) == cli.EXIT_VALIDATION


def test_gen_writes_reference_layout(tmp_path):
    spec = write(tmp_path, "spec.json", {"dimension": 2, "n0_A": 5, "n0_B": 4, "r": 2,
                                         "seed": 3, "omega_A": [1.0, 2.0],
                                         "omega_B": "zero"})
    out = str(tmp_path / "gen")
    assert cli.main(["gen", "--spec", spec, "--out", out]) == cli.EXIT_OK
    A = cli.read_matrix_market(os.path.join(out, "A.mtx"))
    f = cli.read_dense_array(os.path.join(out, "f.mtx"))
    prob = cli.build_inline_problem(json.loads(open(spec).read()))
    assert (A != prob.A).nnz == 0 and np.array_equal(f, prob.f)
    assert A.shape == (25, 25) and f.shape == (25, 2)


def test_named_omegas_and_errors():
    assert cli.resolve_omega("zero") is None
    assert len(cli.resolve_omega("example2_A")) == 3
    assert cli.resolve_omega([1, 2]) == (1.0, 2.0)
    with pytest.raises(ValueError):
        cli.resolve_omega("nope")


def test_matrix_market_rejects_dense_and_complex(tmp_path):
    p = str(tmp_path / "d.mtx")
    cli.write_dense_array(np.ones((3, 2)), p)
    with pytest.raises(cli.SparseFormatError):
        cli.read_matrix_market(p)


def test_factor_roundtrip(tmp_path):
    from paper_2312_02891_b200 import LowRankSolution
    rng = np.random.default_rng(0)
    Z = rng.standard_normal((7, 4)) + 1j * rng.standard_normal((7, 4))
    Y = rng.standard_normal((5, 4)) + 1j * rng.standard_normal((5, 4))
    sol = LowRankSolution(Z=Z, gammas=[1 + 2j, -3.0], Y=Y, r=2)
    cli.save_solution(sol, str(tmp_path))
    back = cli.load_solution(str(tmp_path), r=2)
    assert np.array_equal(back.Z, Z) and np.array_equal(back.Y, Y)
    assert np.array_equal(back.gamma_diag(), sol.gamma_diag())
