"""The native ADI outer loop (sad_adi_run) against the Python loop it replaces
(DeviceAdi._run_python) and the oracle's golden records: same steps, same
inner counts (+-2), same residual history."""

import os
import warnings

import numpy as np
import pytest

from paper_2312_02891_b200 import configs as cfgs

from conftest import GOLD, read_steps_csv

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _engine(name, **kw):
    import paper_2312_02891_b200 as pb
    spec = cfgs.CONFIGS[name]
    A, B, M, C, f, g = cfgs.build_problem(name)
    pairs, cyclic = spec.load_shift_pairs()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
    strategy = kw.pop("strategy", spec.strategy)
    cfg = pb.AdiConfig(strategy=strategy, kmax=kw.pop("kmax", spec.kmax),
                       outer_tolerance=spec.outer_tolerance, gap_budget=kw.pop("gap_budget", None),
                       precond_kind_A="jacobi", precond_kind_B="jacobi")
    seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
    return pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible, **kw)


@pytest.mark.parametrize("name", ["c1", "c2", "c3s", "c5s"])
@pytest.mark.parametrize("concurrent", [True, False])
def test_native_loop_matches_python_loop(name, concurrent):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        eng = _engine(name, concurrent=concurrent)
        assert eng.native
        sol_n, rep_n, st_n = eng.run()
        sol_p, rep_p, st_p = eng._run_python()
    assert rep_n.outer_iterations == rep_p.outer_iterations
    assert rep_n.converged == rep_p.converged
    for a, b in zip(rep_n.records, rep_p.records):
        assert abs(a.inner_it_A - b.inner_it_A) <= 2 and abs(a.inner_it_B - b.inner_it_B) <= 2
        assert abs(a.scaled_res - b.scaled_res) <= 1e-6 * b.scaled_res
        assert abs(a.delta_A - b.delta_A) <= 1e-6 * b.delta_A
        assert abs(a.u - b.u) <= 1e-6 * max(b.u, 1e-300)
    Zn, Zp = sol_n.Z, sol_p.Z
    gn = np.repeat(sol_n.gammas, sol_n.r)
    rel = np.linalg.norm((Zn - Zp) * gn) / np.linalg.norm(Zp * gn)
    assert rel < 1e-6


def test_native_loop_c1_matches_golden():
    gold = read_steps_csv(os.path.join(GOLD, "oracle_c1_gmres.csv"))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        sol, rep, _ = _engine("c1").run()
    assert rep.converged and rep.outer_iterations == len(gold)
    for rec, gd in zip(rep.records, gold):
        assert abs(rec.inner_it_A - gd["inner_it_A"]) <= 2
        assert abs(rec.inner_it_B - gd["inner_it_B"]) <= 2


@pytest.mark.parametrize("strategy", ["fixed", "dynamic_mid", "dynamic_b", "dynamic_b_bl"])
def test_native_loop_strategies(strategy):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        eng = _engine("c1", strategy=strategy)
        _, rep_n, _ = eng.run()
        _, rep_p, _ = eng._run_python()
    assert rep_n.outer_iterations == rep_p.outer_iterations
    for a, b in zip(rep_n.records, rep_p.records):
        assert abs(a.delta_A - b.delta_A) <= 1e-6 * b.delta_A
        assert abs(a.delta_B - b.delta_B) <= 1e-6 * b.delta_B
        assert a.clamped_A_min == b.clamped_A_min and a.clamped_B_min == b.clamped_B_min


def test_native_gram_algebra_r_gt_2():
    """r > 2 takes the Jacobi eigensolver path: config 3s (r = 3)."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        eng = _engine("c3s", concurrent=False)
        _, rep_n, _ = eng.run()
        _, rep_p, _ = eng._run_python()
    assert eng.problem.r == 3
    for a, b in zip(rep_n.records, rep_p.records):
        assert abs(a.achieved_rA - b.achieved_rA) <= 1e-9 * b.achieved_rA
        assert abs(a.scaled_res - b.scaled_res) <= 1e-6 * b.scaled_res


@pytest.mark.parametrize("gap", [0.0, 3e-7])
def test_native_loop_explicit_gap_budget(gap):
    """AdiConfig.gap_budget is used whenever it is not None (adi.py:563-565): a
    budget of 0.0 is a budget (all tolerances at their lower clamps), not "unset"."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        eng = _engine("c1", kmax=4, gap_budget=gap)
        _, rep_n, _ = eng.run()
        _, rep_p, _ = eng._run_python()
        _, rep_d, _ = _engine("c1", kmax=4).run()
    for a, b, d in zip(rep_n.records, rep_p.records, rep_d.records):
        assert abs(a.delta_A - b.delta_A) <= 1e-6 * b.delta_A
        assert abs(a.delta_B - b.delta_B) <= 1e-6 * b.delta_B
        assert a.delta_A != d.delta_A           # not the default outer_tolerance * ||f g^*||
